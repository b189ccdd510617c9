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
// Kernel structure (224 threads, one CTA per SM, persistent):
//   warps 0, 6 TMA producers (one thread each, alternate k-blocks) over a
//              STAGES-deep smem ring
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
#include <array>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>
#include <cstdio>
#include <cstring>

#include "accudnn_kernels.h"
#include "pdl.cuh"
#include "sm100_ptx.cuh"

namespace accudnn {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 32;
// warp 0 and warps 6.. issue TMA loads (k-block kc by producer kc % kProducers):
// one thread issues a stage every ~240-480 cycles (a TMA instruction blocks
// its issuer ~120-240 cycles), so two issuers keep the ring full
constexpr int kProducers = 2;
constexpr int kThreads = 192 + 32 * (kProducers - 1);
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
  long long* trace;    // debug: per-CTA clock64 stamps (accudnn_conv_trace), or nullptr
  int tma_out;         // epilogue stores through tmC (bulk tensor stores / reduce-adds)
  float* stats;        // FWD: per-32-row column sums / sums of squares [2][ceil(M/32)][Ng]
                       // of the output (the next batch norm's statistics), or nullptr
  int a_packed;        // WGRAD: A stage (4 MN atoms) is one 3-D TMA box
  int b_packed;        // DGRAD: B stage (BN/32 MN atoms) is one 4-D box; WGRAD 1x1: one 3-D box
  // stream-K (single-CTA tiles): CTA c owns the (tile, k-block) iterations
  // [c*T/G, (c+1)*T/G) of the tile-major iteration space T = tiles * kb_total;
  // a tile cut between CTAs leaves one partial per segment in its workspace
  // block and the last-arriving segment sums them in segment order
  // 2-slice split-K reduced in L2: the output is zeroed first and both
  // slices bulk reduce-add their tiles into it; (0 + a) + b == (0 + b) + a
  // bit for bit (one rounding per add, the first exact), so the arrival
  // order does not matter -- no workspace, no reduce kernel
  int pair_add;
  int streamk;
  int sk_maxseg;       // segments per tile at most (workspace blocks per tile)
  unsigned* fix_cnt;   // per-tile arrival counters (zero between launches)
};

// experiment switch (ACCUDNN_CONV_DRAIN=1): epilogues wait for their bulk
// stores' global writes before the CTA exits (default: only for the reads)
__constant__ int g_conv_drain = 0;

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
__device__ __forceinline__ void tma_4d(const CUtensorMap* tm, uint32_t dst, uint64_t* bar, int c0,
                                       int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}
// multicast variants: the box lands at the same smem offset in every CTA of
// `mask` and completes tx bytes on each destination's barrier at `bar`'s offset
__device__ __forceinline__ void tma_2d_mc(const CUtensorMap* tm, uint32_t dst, uint64_t* bar,
                                          int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_3d_mc(const CUtensorMap* tm, uint32_t dst, uint64_t* bar,
                                          int c0, int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_4d_mc(const CUtensorMap* tm, uint32_t dst, uint64_t* bar,
                                          int c0, int c1, int c2, int c3, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3), "h"(mask)
      : "memory");
}
// arrive on `bar` (same offset) in every CTA of `mask` when this thread's
// previously issued tcgen05.mma complete
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(ptx::smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// CTA pair (cta_group::2) loads: the box lands in this CTA's shared memory
// and completes its bytes on the pair leader's barrier (shared::cluster
// address `bar_cl`)
__device__ __forceinline__ void tma_2d_g2(const CUtensorMap* tm, uint32_t dst, uint32_t bar_cl,
                                          int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar_cl), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d_g2(const CUtensorMap* tm, uint32_t dst, uint32_t bar_cl,
                                          int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_4d_g2(const CUtensorMap* tm, uint32_t dst, uint32_t bar_cl,
                                          int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_im2col_g2(const CUtensorMap* tm, uint32_t dst, uint32_t bar_cl,
                                              int c, int w, int h, int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.im2col.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar_cl), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow),
      "h"(oh)
      : "memory");
}
// shared::cluster address of the same shared-memory offset in cluster CTA 0
__device__ __forceinline__ uint32_t mapa_cta0(uint32_t saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cl(uint32_t bar_cl, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(
                   bar_cl),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl)
               : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
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
// smem -> global bulk tensor store (or element-wise add into global), 2-D
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, uint32_t src, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tm)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, uint32_t src, int c0, int c1,
                                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tm)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* tm, uint32_t src, int c0,
                                                  int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tm)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N bulk groups still reading their smem source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// global output row offset (floats) of GEMM row m
// stream-K partition: the CTA whose iteration range [c*T/G, (c+1)*T/G)
// holds iteration x (host and device compute the same)
__host__ __device__ __forceinline__ int sk_cta_of(long long x, long long T, int G) {
  int c = static_cast<int>((x * G) / T);
  while (c + 1 < G && ((c + 1) * T) / G <= x) ++c;
  while (c > 0 && (c * T) / G > x) --c;
  return c;
}

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

// CM = 2: a cluster of two CTAs on adjacent M-tiles of the same N-tile; each
// loads its own A and half of B, multicasting the B half to both (B traffic
// from L2 halves); both MMA warps release a stage on both CTAs
// BS = 1 (B-stationary, split-K 1, CM 1): a CTA keeps one N-tile for all its
// units, loads that tile's whole B (every k-block, <= ~128 KB) into shared
// memory once, and streams only A through the ring -- half the operand
// traffic of a 128 x BN tile for short-K GEMMs (1x1 convolutions)
// G = 2 (CM 2, FWD / DGRAD): the pair runs 2-SM MMAs (tcgen05 cta_group::2,
// 256 x BN tiles): each CTA stages its 128 rows of A and half of the B
// columns, both CTAs' loads complete on the even CTA's barriers, whose MMA
// warp issues for the pair; each CTA's TMEM holds its 128 rows x BN.  Per SM
// and k-block that is 16 KB of A + BN/2 x 128 B of B written and read in
// shared memory instead of 16 KB + BN x 128 B: the stage traffic, which bounds
// the single-CTA k-block rate, halves on the B side
template <int MODE, int BN, int STAGES, int CM, int BS, int G, int SK, int KC>
__global__ void __launch_bounds__(kThreads, 1)
    conv_sm100_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, const Prob a) {
  static_assert(G == 1 || (CM == 2 && BS == 0 && MODE != WGRAD), "2-SM tiles: FWD / DGRAD pairs");
  // KC: split-K across a CTA pair (cluster of 2): CTA rank r accumulates the
  // k-blocks of half r of the tile in its own TMEM; rank 1 ships its
  // accumulator chunk by chunk into rank 0's staging buffers through
  // distributed shared memory, rank 0 adds (slice 0 + slice 1, the fixed
  // order of the workspace reduction) and stores the tile.  No workspace
  // round trip, no reduce kernel, and the pair is co-scheduled by hardware.
  static_assert(!KC || (CM == 1 && BS == 0 && G == 1 && SK == 0 && MODE != WGRAD),
                "K-split pairs: single-CTA FWD / DGRAD tiles");
  constexpr int CLS = CM > 1 ? CM : (KC ? 2 : 1);  // cluster size
  constexpr bool kAmn = (MODE == WGRAD);
  constexpr bool kBmn = (MODE != FWD);
  constexpr uint32_t kABytes = kBM * kBK * 4;
  constexpr uint32_t kBBytes = BN * kBK * 4;
  constexpr uint32_t kBLocal = kBBytes / G;  // this CTA's B bytes per stage
  constexpr uint32_t kStageBytes = BS ? kABytes : kABytes + kBLocal;  // ring stage
  constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  // [ring: STAGES x stage] [BS: B region, kb_total x kBBytes] [barriers] [epilogue staging]
  const uint32_t ring_bytes =
      STAGES * kStageBytes + (BS ? static_cast<uint32_t>(a.kb_total) * kBBytes : 0u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ring_bytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;      // [2] accumulator drained
  uint64_t* bfull = tempty + 2;      // BS: the stationary B tile landed
  uint64_t* kc_full = bfull + 1;     // KC rank 0: [warp][slot] peer chunk landed (32 arrivals)
  uint64_t* kc_empty = kc_full + 8;  // KC rank 1: [warp][slot] rank 0's slot free again
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kc_empty + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 1024 + 768] = gtimer();
  const uint32_t crank = CLS > 1 ? cluster_ctarank() : 0u;
  const int cid = static_cast<int>(blockIdx.x) / CLS;    // cluster index
  const int ncl = static_cast<int>(gridDim.x) / CLS;     // clusters in the grid
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << CM) - 1u);
  // work unit -> (split, m-tile, n-tile); with CM = 2 the unit is a tile pair
  auto decode = [&](int u, int& split, int& tile, int& tm, int& tn) {
    if constexpr (KC) {  // the unit is a tile; the split is the CTA's rank
      split = static_cast<int>(crank);
      tile = u;
      tm = u % a.tiles_m;
      tn = u / a.tiles_m;
      return;
    }
    split = u % a.splits;
    const int pair = u / a.splits;
    if (BS) {  // the grid is a multiple of tiles_n: u % tiles_n is fixed per CTA
      tn = u % a.tiles_n;
      tm = u / a.tiles_n;
      tile = tn * a.tiles_m + tm;
    } else if (CM == 1) {
      tile = pair;
      tm = pair % a.tiles_m;
      tn = pair / a.tiles_m;
    } else {
      const int tiles_m2 = (a.tiles_m + 1) / 2;
      tm = (pair % tiles_m2) * 2 + static_cast<int>(crank);
      tn = pair / tiles_m2;
      tile = tn * a.tiles_m + tm;
    }
  };

  // the work of this CTA as a sequence of segments (tile, k-blocks [kb0, kb1));
  // every role walks the same sequence.  split = the segment's index within
  // its tile, nseg = the tile's segment count (1: the segment is the tile)
  // stream-K is its own instantiation: the tile-sequenced kernels keep the
  // lean loop (the run-time switch cost every launch ~5%, measured)
  static_assert(!SK || (CM == 1 && BS == 0 && G == 1), "stream-K: single-CTA tiles only");
  constexpr bool kSK = SK != 0;
  const long long sk_T = static_cast<long long>(a.tiles_m) * a.tiles_n * a.kb_total;
  auto seg_first = [&]() -> long long {
    return (kSK && a.streamk) ? (static_cast<long long>(cid) * sk_T) / ncl : cid;
  };
  const long long sk_end = (static_cast<long long>(cid) + 1) * sk_T / ncl;
  auto seg_next = [&](long long& pos, int& split, int& tile, int& tm, int& tn, int& kb0, int& kb1,
                      int& nseg) -> bool {
    if (kSK && a.streamk) {
      if (pos >= sk_end) return false;
      tile = static_cast<int>(pos / a.kb_total);
      kb0 = static_cast<int>(pos - static_cast<long long>(tile) * a.kb_total);
      kb1 = static_cast<int>(min(static_cast<long long>(a.kb_total), kb0 + (sk_end - pos)));
      pos += kb1 - kb0;
      tm = tile % a.tiles_m;
      tn = tile / a.tiles_m;
      const long long t0 = static_cast<long long>(tile) * a.kb_total;
      const int cf = sk_cta_of(t0, sk_T, ncl);
      split = cid - cf;
      nseg = sk_cta_of(t0 + a.kb_total - 1, sk_T, ncl) - cf + 1;
      return true;
    }
    if (pos >= a.units) return false;
    decode(static_cast<int>(pos), split, tile, tm, tn);
    kb0 = split * a.kb_per_split;
    kb1 = min(a.kb_total, kb0 + a.kb_per_split);
    nseg = a.splits;
    pos += ncl;
    return true;
  };
  // stream-K fix-up: "this CTA arrived last on the tile" (barrier region)
  volatile int& s_fix_last = *reinterpret_cast<volatile int*>(tmem_slot + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], G == 2 ? 1 : CM);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], G == 2 ? 2 * (kEpiThreads / 32) : kEpiThreads);
    }
    ptx::mbar_init(bfull, 1);
    if (KC)
      for (int i = 0; i < 8; ++i) {
        ptx::mbar_init(&kc_full[i], 1);
        ptx::mbar_init(&kc_empty[i], 1);
      }
    ptx::fence_mbar_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (a.tma_out) prefetch_tmap(&tmC);
  }
  if (warp == 1) {
    if constexpr (G == 2)
      ptx::tmem_alloc_pair<kTmemCols>(tmem_slot);
    else
      ptx::tmem_alloc<kTmemCols>(tmem_slot);
  }
  ptx::tc_fence_before();
  if (CLS > 1)
    cluster_sync_all();  // peers' barriers initialised before any multicast / remote arrive
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t smem_base = ptx::smem_u32(smem);
  // everything above overlapped the previous kernel's tail (PDL)
  pdl_wait();
  if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 1024 + 769] = gtimer();

  if (warp == 0 || warp >= 6) {
    if (lane == 0) {
      // ============================ TMA producers ============================
      const uint32_t pid = warp == 0 ? 0u : static_cast<uint32_t>(warp - 5);
      uint32_t kc = 0;  // k-blocks of this CTA (ring position)
      if (BS && pid == 0 && cid < a.units) {
        // the whole B tile of this CTA's N-tile, every k-block, once
        const int n0 = (cid % a.tiles_n) * BN;
        const uint32_t sBs = smem_base + STAGES * kStageBytes;
        mbar_expect_tx(bfull, static_cast<uint32_t>(a.kb_total) * kBBytes);
        for (int kb = 0; kb < a.kb_total; ++kb) {
          const uint32_t sB = sBs + kb * kBBytes;
          const int kk = kb * kBK;
          if constexpr (MODE == FWD) {
            tma_2d(&tmB, sB, bfull, kk, n0);
          } else if constexpr (MODE == DGRAD) {
            const int t = kk / a.K, co0 = kk - t * a.K;
            const int tr = t / a.Sc, ts = t - tr * a.Sc;
            const int tap = (a.r0 - a.stride * tr) * a.S + (a.s0 - a.stride * ts);
            if (a.b_packed) {
              tma_4d(&tmB, sB, bfull, 0, co0, n0 / 32, tap);
            } else {
#pragma unroll
              for (int b = 0; b < BN / 32; ++b)
                tma_3d(&tmB, sB + b * 4096, bfull, n0 + 32 * b, tap, co0);
            }
          }
        }
      }
      long long pos = seg_first();
      int split, tile, tm, tn, kb0, kb1, nseg;
      while (seg_next(pos, split, tile, tm, tn, kb0, kb1, nseg)) {
        const int m0 = tm * kBM, n0 = tn * BN;
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
          if (kc % kProducers != pid) continue;
          const uint32_t stage = kc % STAGES;
          if (kc >= STAGES) ptx::mbar_wait(&empty[stage], ((kc / STAGES) - 1) & 1);
          if (a.trace && kc < 256) a.trace[blockIdx.x * 1024 + kc] = clock64();
          const uint32_t sA = smem_base + stage * kStageBytes;
          const uint32_t sB = sA + kABytes;
          uint64_t* bar = &full[stage];
          uint32_t full_cl = 0;  // G = 2: the even CTA's barrier
          if constexpr (G == 2) {
            // the even CTA's producer expects both CTAs' bytes; the odd CTA's
            // loads only complete bytes on it
            full_cl = mapa_cta0(ptx::smem_u32(bar));
            if (crank == 0) mbar_expect_tx(bar, 2 * kStageBytes);
          } else {
            mbar_expect_tx(bar, kStageBytes);
          }
          const int kk = kb * kBK;
          if constexpr (G == 2 && MODE == FWD) {
            if (a.a_tiled) {
              tma_2d_g2(&tmA, sA, full_cl, kk, m0);
            } else {
              const int tap = kk / a.C, c0 = kk - tap * a.C;
              const int r = tap / a.S, s = tap - r * a.S;
              tma_im2col_g2(&tmA, sA, full_cl, c0, pj * a.stride - a.pad, pi * a.stride - a.pad, pn,
                            static_cast<uint16_t>(s), static_cast<uint16_t>(r));
            }
            tma_2d_g2(&tmB, sB, full_cl, kk, n0 + static_cast<int>(crank) * (BN / 2));
          } else if constexpr (G == 2 && MODE == DGRAD) {
            const int t = kk / a.K, co0 = kk - t * a.K;
            const int tr = t / a.Sc, ts = t - tr * a.Sc;
            const int tap = (a.r0 - a.stride * tr) * a.S + (a.s0 - a.stride * ts);
            if (a.a_tiled) {
              tma_2d_g2(&tmA, sA, full_cl, co0, m0);
            } else {
              tma_im2col_g2(&tmA, sA, full_cl, co0, pj + a.lo_w, pi + a.lo_h, pn,
                            static_cast<uint16_t>(ts), static_cast<uint16_t>(tr));
            }
            constexpr int kHalf = BN / 64;  // this CTA's 32-column atoms
            const int b0 = static_cast<int>(crank) * kHalf;
            if (a.b_packed) {
              tma_4d_g2(&tmB, sB, full_cl, 0, co0, n0 / 32 + b0, tap);
            } else {
#pragma unroll
              for (int b = 0; b < kHalf; ++b)
                tma_3d_g2(&tmB, sB + b * 4096, full_cl, n0 + 32 * (b0 + b), tap, co0);
            }
          } else if constexpr (BS && MODE == FWD) {  // A only
            if (a.a_tiled) {
              tma_2d(&tmA, sA, bar, kk, m0);
            } else {
              const int tap = kk / a.C, c0 = kk - tap * a.C;
              const int r = tap / a.S, s = tap - r * a.S;
              tma_im2col(&tmA, sA, bar, c0, pj * a.stride - a.pad, pi * a.stride - a.pad, pn,
                         static_cast<uint16_t>(s), static_cast<uint16_t>(r));
            }
          } else if constexpr (BS && MODE == DGRAD) {
            const int t = kk / a.K, co0 = kk - t * a.K;
            const int tr = t / a.Sc, ts = t - tr * a.Sc;
            if (a.a_tiled) {
              tma_2d(&tmA, sA, bar, co0, m0);
            } else {
              tma_im2col(&tmA, sA, bar, co0, pj + a.lo_w, pi + a.lo_h, pn,
                         static_cast<uint16_t>(ts), static_cast<uint16_t>(tr));
            }
          } else if constexpr (MODE == FWD) {
            if (a.a_tiled) {
              tma_2d(&tmA, sA, bar, kk, m0);
            } else {
              const int tap = kk / a.C, c0 = kk - tap * a.C;
              const int r = tap / a.S, s = tap - r * a.S;
              tma_im2col(&tmA, sA, bar, c0, pj * a.stride - a.pad, pi * a.stride - a.pad, pn,
                         static_cast<uint16_t>(s), static_cast<uint16_t>(r));
            }
            if (CM > 1)
              tma_2d_mc(&tmB, sB + crank * (kBBytes / CM), bar, kk,
                        n0 + static_cast<int>(crank) * (BN / CM), kMask);
            else
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
            if (CM > 1) {  // this CTA's half of the atoms, multicast to the pair
              constexpr int kHalf = BN / 32 / CM;
              const int b0 = static_cast<int>(crank) * kHalf;
              if (a.b_packed) {
                tma_4d_mc(&tmB, sB + b0 * 4096, bar, 0, co0, n0 / 32 + b0, tap, kMask);
              } else {
#pragma unroll
                for (int b = 0; b < kHalf; ++b)
                  tma_3d_mc(&tmB, sB + (b0 + b) * 4096, bar, n0 + 32 * (b0 + b), tap, co0, kMask);
              }
            } else if (a.b_packed) {  // {ci 32, co, ci-block, tap}: all BN/32 atoms at once
              tma_4d(&tmB, sB, bar, 0, co0, n0 / 32, tap);
            } else {
#pragma unroll
              for (int b = 0; b < BN / 32; ++b)
                tma_3d(&tmB, sB + b * 4096, bar, n0 + 32 * b, tap, co0);
            }
          } else {
            if (a.a_packed) {  // {co 32, pixel, co-block}: the 4 atoms of the stage at once
              tma_3d(&tmA, sA, bar, 0, kk, m0 / 32);
            } else {
#pragma unroll
              for (int b = 0; b < kBM / 32; ++b) tma_2d(&tmA, sA + b * 4096, bar, m0 + 32 * b, kk);
            }
            if (a.b_packed) {  // 1x1 stride 1: {ci 32, pixel, ci-block}
              tma_3d(&tmB, sB, bar, 0, kk, n0 / 32);
            } else {
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
    }
  } else if (warp == 1) {
    if (lane == 0 && (G == 1 || crank == 0)) {
      // ============================ MMA issuer ============================
      constexpr uint32_t idesc = ptx::idesc_tf32(kBM * G, BN, kAmn, kBmn);
      uint32_t kc = 0;
      int j = 0;  // units processed by this CTA
      if (BS && cid < a.units) ptx::mbar_wait(bfull, 0);
      long long pos = seg_first();
      int split, tile, tm, tn, kb0, kb1, nseg;
      for (; seg_next(pos, split, tile, tm, tn, kb0, kb1, nseg); ++j) {
        const int acc = j & 1;
        if (j >= 2) ptx::mbar_wait(&tempty[acc], ((j >> 1) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + static_cast<uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++kc) {
          const uint32_t stage = kc % STAGES;
          ptx::mbar_wait(&full[stage], (kc / STAGES) & 1);
          if (a.trace && kc < 256) a.trace[blockIdx.x * 1024 + 256 + kc] = clock64();
          ptx::tc_fence_after();
          const uint32_t sA = smem_base + stage * kStageBytes;
          const uint32_t sB = BS ? smem_base + STAGES * kStageBytes + kb * kBBytes : sA + kABytes;
#pragma unroll
          for (int ks = 0; ks < kBK / 8; ++ks) {
            const uint64_t ad = kAmn ? ptx::smem_desc(sA + ks * 1024, 4096, 512, 1)
                                     : ptx::smem_desc(sA + ks * 32, 16, 1024, 2);
            const uint64_t bd = kBmn ? ptx::smem_desc(sB + ks * 1024, 4096, 512, 1)
                                     : ptx::smem_desc(sB + ks * 32, 16, 1024, 2);
            if constexpr (G == 2)
              ptx::mma_tf32_pair(d_tmem, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
            else
              ptx::mma_tf32(d_tmem, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
          }
          if (G == 2)
            ptx::mma_commit_pair(&empty[stage], kMask);  // both CTAs' stages consumed
          else if (CM > 1)
            mma_commit_mc(&empty[stage], kMask);  // the stage holds the peer's B half too
          else
            ptx::mma_commit(&empty[stage]);
        }
        if (G == 2)
          ptx::mma_commit_pair(&tfull[acc], kMask);  // both CTAs' accumulator rows
        else
          ptx::mma_commit(&tfull[acc]);
      }
    }
    // (PDL) the CTA's tensor-core work is issued: its successor may be
    // scheduled while the last epilogue drains (it still waits for this grid)
    if (lane == 0) pdl_trigger();
  } else {
    // ============================ epilogue ============================
    // Each warp drains its TMEM lane quadrant (32 rows) in 32-column chunks.
    // TMA-store path (row-major outputs and split-K slices): tcgen05.ld ->
    // registers -> one of two 4 KB smem buffers in the SWIZZLE_128B layout
    // -> one bulk tensor store (or element-wise add for beta = 1) issued by
    // lane 0, which completes asynchronously while the next chunk is
    // staged in the other buffer.  Scatter outputs (strided dgrad classes) use coalesced
    // 128-byte row segments from the same smem transpose instead.
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int ew = warp - 2;    // staging buffers of this warp
    float* stage_buf = reinterpret_cast<float*>(smem + ring_bytes + 1024) + ew * 2048;
    const uint32_t sbuf0 = ptx::smem_u32(stage_buf);
    // KC: rank 0's receive slots [warp][2] x 4 KB, after the staging buffers
    const uint32_t recv0 = ptx::smem_u32(smem + ring_bytes + 1024 + 4 * 8192);
    const int rr_lo = lane >> 3;  // read-back row within a group of 4 (scatter path)
    const int gg = lane & 7;      // read-back 16-byte granule
    uint32_t nchunk = 0;          // chunks staged by this warp (buffer parity)
    int j = 0;
    long long pos = seg_first();
    int split, tile, tm, tn, kb0, kb1, nseg;
    for (; seg_next(pos, split, tile, tm, tn, kb0, kb1, nseg); ++j) {
      const int m0 = tm * kBM + quad * 32, n0 = tn * BN;
      const int acc = j & 1;
      ptx::mbar_wait(&tfull[acc], (j >> 1) & 1);
      if (a.trace && threadIdx.x == 64 && j < 128) a.trace[blockIdx.x * 1024 + 512 + 2 * j] = clock64();
      ptx::tc_fence_after();
      const uint32_t trow = tmem + static_cast<uint32_t>(acc * BN) +
                            (static_cast<uint32_t>(quad * 32) << 16);
      const int ncols = min(BN, a.Ng - n0);  // multiple of 4
      const bool partial = nseg > 1 && !KC && !a.pair_add;
      // stream-K partial: plain stores into the segment's workspace block
      // [128][BN] (the tile's other segments may still be running)
      const bool skp = kSK && a.streamk && partial;
      float* sk_blk = skp ? a.ws + (static_cast<long long>(tile) * a.sk_maxseg + split) * (kBM * BN)
                          : nullptr;
      const int nch = (ncols + 31) / 32;
#pragma unroll 1
      for (int ci = 0; ci < nch; ++ci) {
        const int c0 = ci * 32;
        float cur[32];
        ptx::tmem_ld32(trow + c0, cur);
        if (ci + 1 >= nch) {  // accumulator drained: release it to the MMA warp
          ptx::tc_fence_before();
          if constexpr (G == 2) {  // one arrive per warp on the even CTA's barrier
            __syncwarp();
            if (lane == 0) mbar_arrive_cl(mapa_cta0(ptx::smem_u32(&tempty[acc])));
          } else {
            ptx::mbar_arrive(&tempty[acc]);
          }
        }
        const uint32_t sbuf = sbuf0 + (nchunk & 1) * 4096;
        if constexpr (KC) {
          // chunk hand-off: rank 1 stages its chunk in its own buffer `sbuf`
          // and one bulk copy (TMA engine, DSMEM) moves it into rank 0's
          // receive slot (warp, chunk parity), completing on rank 0's
          // kc_full; rank 0 frees the slot (kc_empty, remote arrive) as soon
          // as it has the values in registers, adds its own chunk and stores.
          // Use u >= 1 of a slot waits for the u-th kc_empty arrival.
          const int slot = quad * 2 + static_cast<int>(nchunk & 1);
          const uint32_t use = nchunk >> 1;
          const uint32_t rslot = recv0 + static_cast<uint32_t>(slot) * 4096;
          if (crank == 1) {
            if (use >= 1) ptx::mbar_wait_acq_cluster(&kc_empty[slot], (use - 1) & 1);
            if (lane == 0) bulk_wait_read<1>();  // our copy out of this buffer has read it
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 8; ++g)
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                               sbuf + lane * 128 + ((g ^ (lane & 7)) << 4)),
                           "f"(cur[4 * g]), "f"(cur[4 * g + 1]), "f"(cur[4 * g + 2]),
                           "f"(cur[4 * g + 3])
                           : "memory");
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              uint32_t rbuf, rbar;
              asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rbuf) : "r"(rslot));
              asm volatile("mapa.shared::cluster.u32 %0, %1, 0;"
                           : "=r"(rbar)
                           : "r"(ptx::smem_u32(&kc_full[slot])));
              asm volatile(
                  "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes"
                  " [%0], [%1], 4096, [%2];" ::"r"(rbuf),
                  "r"(sbuf), "r"(rbar)
                  : "memory");
              bulk_commit();
            }
            ++nchunk;
            continue;
          }
          if (lane == 0) mbar_expect_tx(&kc_full[slot], 4096);  // arm this use
          ptx::mbar_wait(&kc_full[slot], use & 1);
          float peer[32];
#pragma unroll
          for (int g = 0; g < 8; ++g)
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(peer[4 * g]), "=f"(peer[4 * g + 1]), "=f"(peer[4 * g + 2]),
                           "=f"(peer[4 * g + 3])
                         : "r"(rslot + lane * 128 + ((g ^ (lane & 7)) << 4))
                         : "memory");
          __syncwarp();
          if (lane == 0) {  // the slot's values are in registers: hand it back
            uint32_t pe;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 1;"
                         : "=r"(pe)
                         : "r"(ptx::smem_u32(&kc_empty[slot])));
            mbar_arrive_cl(pe);
            bulk_wait_read<1>();  // our store that used `sbuf` has read it
          }
          __syncwarp();
#pragma unroll
          for (int g = 0; g < 32; ++g) cur[g] += peer[g];  // slice 0 + slice 1
#pragma unroll
          for (int g = 0; g < 8; ++g)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                             sbuf + lane * 128 + ((g ^ (lane & 7)) << 4)),
                         "f"(cur[4 * g]), "f"(cur[4 * g + 1]), "f"(cur[4 * g + 2]),
                         "f"(cur[4 * g + 3])
                         : "memory");
        } else {
        if (lane == 0) bulk_wait_read<1>();  // the store that used this buffer has read it
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 8; ++g)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                           sbuf + lane * 128 + ((g ^ (lane & 7)) << 4)),
                       "f"(cur[4 * g]), "f"(cur[4 * g + 1]), "f"(cur[4 * g + 2]), "f"(cur[4 * g + 3])
                       : "memory");
        }
        if (a.stats && !partial) {
          // column sums of this 32x32 chunk for the next batch norm: lane l
          // walks column l of the staged (swizzled) chunk; rows past M skipped
          __syncwarp();
          const int col = n0 + c0 + lane;
          float cs = 0.f, cq = 0.f;
          const int nrows = min(32, a.M - m0);
#pragma unroll 8
          for (int r = 0; r < nrows; ++r) {
            float v;
            asm volatile("ld.shared.f32 %0, [%1];"
                         : "=f"(v)
                         : "r"(sbuf + r * 128 + ((((lane >> 2) ^ (r & 7))) << 4) + (lane & 3) * 4));
            cs += v;
            cq += v * v;
          }
          if (nrows > 0 && col < a.Ng) {
            const long long P = (a.M + 31) / 32;
            const long long slot = m0 / 32;
            a.stats[slot * a.Ng + col] = cs;
            a.stats[(P + slot) * a.Ng + col] = cq;
          }
        }
        if (a.tma_out && !skp) {
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (partial)
              tma_store_3d(&tmC, sbuf, n0 + c0, m0, split);
            else if (a.beta || a.pair_add)
              tma_reduce_add_2d(&tmC, sbuf, n0 + c0, m0);
            else
              tma_store_2d(&tmC, sbuf, n0 + c0, m0);
            bulk_commit();
          }
        } else {
          __syncwarp();
          const int col = n0 + c0 + gg * 4;
          const bool col_ok = c0 + gg * 4 < ncols;
          // the 8 rows' destinations (and, accumulating, their old values)
          // first: the loads are independent and all in flight at once (a
          // load -> add -> store chain per row would pay one memory latency
          // per row, ~30 us per 128 x 128 tile)
          float4* d4s[8];
          float4 olds[8];
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int m = m0 + it * 4 + rr_lo;
            d4s[it] = nullptr;
            if (col_ok && m < a.M)
              d4s[it] = reinterpret_cast<float4*>(
                  skp       ? sk_blk + (m - tm * kBM) * BN + (col - n0)
                  : partial ? a.ws + (static_cast<long long>(split) * a.M + m) * a.Ng + col
                            : a.out + out_row(a, m) + col);
            olds[it] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (d4s[it] && a.beta && !partial) olds[it] = __ldcg(d4s[it]);
          }
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rr = it * 4 + rr_lo;
            float4 o;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(o.x), "=f"(o.y), "=f"(o.z), "=f"(o.w)
                         : "r"(sbuf + rr * 128 + ((gg ^ (rr & 7)) << 4)));
            if (d4s[it]) {
              if (a.beta && !partial) {
                o.x += olds[it].x;
                o.y += olds[it].y;
                o.z += olds[it].z;
                o.w += olds[it].w;
              }
              __stcg(d4s[it], o);
            }
          }
        }
        ++nchunk;
      }
      if (nch == 0) {  // tile entirely past Ng (cannot happen with tiles_n = ceil(Ng/BN))
        ptx::tc_fence_before();
        if constexpr (G == 2) {
          __syncwarp();
          if (lane == 0) mbar_arrive_cl(mapa_cta0(ptx::smem_u32(&tempty[acc])));
        } else {
          ptx::mbar_arrive(&tempty[acc]);
        }
      }
      if (kSK && skp) {
        // ---- stream-K fix-up: arrive on the tile; the last segment to
        // arrive sums the tile's partial blocks in segment order (slot 0 is
        // the lowest k-blocks), adds the old output for beta = 1 and stores.
        // Nobody waits for anybody: no assumption about co-resident CTAs.
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64)
          s_fix_last = atomicAdd(a.fix_cnt + tile, 1u) == static_cast<unsigned>(nseg - 1) ? 1 : 0;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (s_fix_last) {
          __threadfence();
          const float* blk0 = a.ws + static_cast<long long>(tile) * a.sk_maxseg * (kBM * BN);
          const int nc4 = ncols >> 2;
          const int rows = min(kBM, a.M - tm * kBM);
          const int total = rows * (BN / 4);
          const int et = threadIdx.x - 64;  // 0..127
          for (int base = et; base < total; base += 128 * 8) {
            float4 o[8];
            int off[8];
            bool ok[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int f = base + e * 128;
              const int r = f / (BN / 4), c4 = f - r * (BN / 4);
              ok[e] = f < total && c4 < nc4;
              off[e] = r * BN + c4 * 4;
              o[e] = ok[e] ? __ldcg(reinterpret_cast<const float4*>(blk0 + off[e]))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (int sl = 1; sl < nseg; ++sl) {
              const float* blk = blk0 + static_cast<long long>(sl) * (kBM * BN);
              float4 p[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)
                p[e] = ok[e] ? __ldcg(reinterpret_cast<const float4*>(blk + off[e]))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                o[e].x += p[e].x;
                o[e].y += p[e].y;
                o[e].z += p[e].z;
                o[e].w += p[e].w;
              }
            }
            float4* d[8];
            float4 old[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int r = off[e] / BN;
              d[e] = ok[e] ? reinterpret_cast<float4*>(a.out + out_row(a, tm * kBM + r) + n0 +
                                                       (off[e] - r * BN))
                           : nullptr;
              if (d[e] && a.beta) old[e] = __ldcg(d[e]);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (d[e]) {
                if (a.beta) {
                  o[e].x += old[e].x;
                  o[e].y += old[e].y;
                  o[e].z += old[e].z;
                  o[e].w += old[e].w;
                }
                __stcg(d[e], o[e]);
              }
          }
          if (threadIdx.x == 64) a.fix_cnt[tile] = 0u;  // every segment has arrived
        }
      }
      if (a.trace && threadIdx.x == 64 && j < 128) a.trace[blockIdx.x * 1024 + 513 + 2 * j] = clock64();
    }
    // the staging buffers must have been read before the CTA retires; the
    // global writes themselves complete with the grid (no need to hold the SM)
    if (lane == 0) {
      if (g_conv_drain)
        bulk_wait_all();
      else
        bulk_wait_read<0>();
    }
  }

  ptx::tc_fence_before();
  if (CLS > 1)
    cluster_sync_all();  // no CTA leaves while its peer may still write / arrive into it
  else
    __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if constexpr (G == 2)
      ptx::tmem_dealloc_pair<kTmemCols>(tmem);
    else
      ptx::tmem_dealloc<kTmemCols>(tmem);
  }
  if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 1024 + 770] = gtimer();
}

// Strided dgrad: zero the input-gradient pixels of the parity classes that
// receive no filter tap (row parity bit in row_empty, column parity in
// col_empty); the classes with taps are written by their GEMMs
__global__ void __launch_bounds__(256) dgrad_zero_empty_kernel(float4* __restrict__ dx, int n,
                                                              int h, int w, int c4, int s,
                                                              unsigned row_empty,
                                                              unsigned col_empty) {
  pdl_wait();
  pdl_trigger();
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  const int row4 = w * c4;
  for (long long row = blockIdx.x; row < static_cast<long long>(n) * h; row += gridDim.x) {
    const int y = static_cast<int>(row % h);
    float4* p = dx + row * row4;
    if ((row_empty >> (y % s)) & 1u) {  // the whole image row
      for (int i = threadIdx.x; i < row4; i += 256) __stcs(p + i, z);
    } else {  // the pixels of the empty column classes
      for (int i = threadIdx.x; i < row4; i += 256)
        if ((col_empty >> ((i / c4) % s)) & 1u) __stcs(p + i, z);
    }
  }
}

// Deterministic split-K reduction: out[map(m)][n] (+)= sum_{s=0..S-1} ws[s][m][n],
// slices always summed in slice order.  One float4 per thread-iteration,
// grid-stride over the M x Ng/4 output vectors (coalesced rows).
__global__ void __launch_bounds__(256) conv_splitk_reduce_kernel(const Prob a) {
  pdl_wait();
  pdl_trigger();
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 148) a.trace[blockIdx.x * 1024 + 771] = gtimer();
  const int ng4 = a.Ng >> 2;
  const long long total = static_cast<long long>(a.M) * ng4;
  const long long slice = static_cast<long long>(a.M) * a.Ng;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * 256) {
    const int m = static_cast<int>(i / ng4);
    const int c = static_cast<int>(i - static_cast<long long>(m) * ng4) * 4;
    const float* src = a.ws + static_cast<long long>(m) * a.Ng + c;
    float4 o = __ldcg(reinterpret_cast<const float4*>(src));
    for (int s0 = 1; s0 < a.splits; s0 += 8) {  // 8 slices in flight, summed in order
      float4 p[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < a.splits) p[u] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + u) * slice));
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < a.splits) {
          o.x += p[u].x;
          o.y += p[u].y;
          o.z += p[u].z;
          o.w += p[u].w;
        }
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

// split-K reduction that also produces the batch-norm column statistics of
// the output.  Block = 32 rows x 32 columns (thread = row x float4): slices
// summed in order per element, then the column sums over the 32 rows in a
// fixed smem order -> one [2][P][Ng] partial slot per (32-row block, column).
// Many slices (the weight gradients' long-K GEMMs: 16-128 slices of a small
// output): a group of 8 lanes per output float4, lane g summing slices
// g, g+8, ... in order (all loads of a lane in flight at once), then a fixed
// xor-shuffle tree over the group -- one memory round trip instead of
// splits/8 sequential ones, and still the same order on every run.
__global__ void __launch_bounds__(256) conv_splitk_reduce_wide_kernel(const Prob a) {
  pdl_wait();
  pdl_trigger();
  const int ng4 = a.Ng >> 2;
  const long long total = static_cast<long long>(a.M) * ng4;
  const long long slice = static_cast<long long>(a.M) * a.Ng;
  const int g = threadIdx.x & 7;
  for (long long i = (blockIdx.x * 256LL + threadIdx.x) >> 3; i < total;
       i += static_cast<long long>(gridDim.x) * 32) {
    const int m = static_cast<int>(i / ng4);
    const int c = static_cast<int>(i - static_cast<long long>(m) * ng4) * 4;
    const float* src = a.ws + static_cast<long long>(m) * a.Ng + c;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = g; s0 < a.splits; s0 += 64) {
      float4 p[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + 8 * u < a.splits)
          p[u] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + 8 * u) * slice));
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + 8 * u < a.splits) {
          o.x += p[u].x;
          o.y += p[u].y;
          o.z += p[u].z;
          o.w += p[u].w;
        }
    }
    // the 8 lanes of this group (groups of a warp may leave the loop apart)
    const unsigned gmask = 0xFFu << (threadIdx.x & 24);
#pragma unroll
    for (int off = 1; off < 8; off <<= 1) {
      o.x += __shfl_xor_sync(gmask, o.x, off, 8);
      o.y += __shfl_xor_sync(gmask, o.y, off, 8);
      o.z += __shfl_xor_sync(gmask, o.z, off, 8);
      o.w += __shfl_xor_sync(gmask, o.w, off, 8);
    }
    if (g == 0) {
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
}

__global__ void __launch_bounds__(256) conv_splitk_reduce_stats_kernel(const Prob a) {
  pdl_wait();
  pdl_trigger();
  __shared__ float4 red1[32][8], red2[32][8];
  const int cbs = a.Ng / 32;
  const long long P = (a.M + 31) / 32;
  const long long slice = static_cast<long long>(a.M) * a.Ng;
  const int tr = threadIdx.x >> 3, tc = threadIdx.x & 7;
  for (long long blk = blockIdx.x; blk < P * cbs; blk += gridDim.x) {
    const long long pb = blk / cbs;
    const int c = static_cast<int>(blk - pb * cbs) * 32 + tc * 4;
    const long long m = pb * 32 + tr;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (m < a.M) {
      const float* src = a.ws + m * a.Ng + c;
      o = __ldcg(reinterpret_cast<const float4*>(src));
      for (int s0 = 1; s0 < a.splits; s0 += 8) {
        float4 p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (s0 + u < a.splits) p[u] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + u) * slice));
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (s0 + u < a.splits) {
            o.x += p[u].x;
            o.y += p[u].y;
            o.z += p[u].z;
            o.w += p[u].w;
          }
      }
      *reinterpret_cast<float4*>(a.out + m * a.Ng + c) = o;
    }
    red1[tr][tc] = o;
    red2[tr][tc] = make_float4(o.x * o.x, o.y * o.y, o.z * o.z, o.w * o.w);
    __syncthreads();
    if (threadIdx.x < 8) {  // column group tc = threadIdx.x, rows in order
      float4 s1 = make_float4(0.f, 0.f, 0.f, 0.f), s2 = s1;
      for (int r = 0; r < 32; ++r) {
        const float4 u = red1[r][threadIdx.x], v = red2[r][threadIdx.x];
        s1.x += u.x; s1.y += u.y; s1.z += u.z; s1.w += u.w;
        s2.x += v.x; s2.y += v.y; s2.z += v.z; s2.w += v.w;
      }
      const int cc = static_cast<int>(blk - pb * cbs) * 32 + threadIdx.x * 4;
      *reinterpret_cast<float4*>(a.stats + pb * a.Ng + cc) = s1;
      *reinterpret_cast<float4*>(a.stats + (P + pb) * a.Ng + cc) = s2;
    }
    __syncthreads();
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
// per-stream workspaces (a concurrent weight-gradient stream must not share
// the compute stream's split-K partials); the entry points select the one
// of their stream before any split-K decision
struct StreamWs {
  cudaStream_t st = nullptr;
  Workspace w;
  int max_ctas = 0;  // persistent grids on this stream use at most this many SMs (0: all)
};
// one entry per registered stream (executors register their weight-gradient
// stream); entries are heap nodes so g_cur stays valid while others come and go
std::vector<std::unique_ptr<StreamWs>> g_stream_ws;
Workspace* g_cur = &g_ws;
int g_cur_ctas = 0;
int cta_slots() { return g_cur_ctas > 0 ? std::min(g_cur_ctas, sm_count()) : sm_count(); }
long long* g_trace = nullptr;  // debug stamps, see accudnn_conv_trace

// the last kFixBytes of every workspace hold the stream-K per-tile arrival
// counters (zeroed when the workspace is set, left zero by every launch)
constexpr size_t kFixBytes = 64 * 1024;
constexpr int kMaxFixTiles = static_cast<int>(kFixBytes / sizeof(unsigned));
size_t usable(size_t bytes) { return bytes > 2 * kFixBytes ? bytes - kFixBytes : 0; }
unsigned* fix_counters(const Workspace& w) {
  return w.ws && usable(w.bytes)
             ? reinterpret_cast<unsigned*>(reinterpret_cast<char*>(w.ws) + w.bytes - kFixBytes)
             : nullptr;
}
void zero_fix_counters(const Workspace& w) {
  if (unsigned* c = fix_counters(w)) {
    cudaMemset(c, 0, kFixBytes);
    cudaDeviceSynchronize();
  }
}
// lazily owned workspace when the caller did not provide one
size_t default_ws_capacity() {
  if (!g_ws.ws && !g_ws.bytes && g_ws_default) {
    if (cudaMalloc(&g_ws.ws, g_ws_default) == cudaSuccess) {
      g_ws.bytes = g_ws_default;
      g_ws.owned = true;
      zero_fix_counters(g_ws);
    } else {
      cudaGetLastError();
      g_ws.ws = nullptr;
    }
  }
  return g_ws.ws ? g_ws.bytes : 0;
}
size_t ws_capacity() { return usable(g_cur == &g_ws ? default_ws_capacity() : g_cur->bytes); }

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

template <int MODE, int BN, int STAGES, int CM, int BS, int G, int SK = 0, int KC = 0>
int launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const Prob& a,
             cudaStream_t st) {
  const size_t ring = BS ? STAGES * kBM * kBK * 4 + static_cast<size_t>(a.kb_total) * BN * kBK * 4
                         : STAGES * (kBM + BN / G) * kBK * 4;
  const size_t smem = ring + 1024 + 1024 + 4 * 8192 + (KC ? 4 * 8192 : 0);
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(conv_sm100_kernel<MODE, BN, STAGES, CM, BS, G, SK, KC>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               227 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
    configured = true;
  }
  if (smem > 227 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  constexpr int CLS = CM > 1 ? CM : (KC ? 2 : 1);
  int grid = CLS * static_cast<int>(std::min<long long>(a.units, cta_slots() / CLS));
  if (BS) grid = std::min(cta_slots(), a.units) / a.tiles_n * a.tiles_n;  // fixed N-tile per CTA
  if (grid < 1) return static_cast<int>(cudaErrorInvalidValue);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CLS;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CLS > 1 ? 2 : 1;
  cudaError_t e =
      cudaLaunchKernelEx(&cfg, conv_sm100_kernel<MODE, BN, STAGES, CM, BS, G, SK, KC>, ta, tb, tc, a);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess || a.splits == 1 || KC || a.pair_add) return static_cast<int>(e);
  if (a.stats) {
    const long long blocks = (static_cast<long long>(a.M) + 31) / 32 * (a.Ng / 32);
    const int rgrid = static_cast<int>(std::min<long long>(blocks, 16LL * sm_count()));
    launch_pdl(conv_splitk_reduce_stats_kernel, rgrid, 256, 0, st, a);
    return static_cast<int>(cudaGetLastError());
  }
  const long long vec = static_cast<long long>(a.M) * (a.Ng / 4);
  static const int wide_from = [] {  // ACCUDNN_REDUCE_WIDE: slices from which 8 lanes share a vector
    const char* e = std::getenv("ACCUDNN_REDUCE_WIDE");
    return e ? std::atoi(e) : 16;
  }();
  if (a.splits >= wide_from) {  // 8 lanes per output vector
    const int wgrid = static_cast<int>(std::min<long long>((vec * 8 + 255) / 256, 16LL * sm_count()));
    launch_pdl(conv_splitk_reduce_wide_kernel, wgrid, 256, 0, st, a);
    return static_cast<int>(cudaGetLastError());
  }
  const int rgrid = static_cast<int>(std::min<long long>((vec + 255) / 256, 8LL * sm_count()));
  launch_pdl(conv_splitk_reduce_kernel, rgrid, 256, 0, st, a);
  return static_cast<int>(cudaGetLastError());
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

// ---- one GEMM of a convolution, re-launchable with any (BN, splits) -------------
struct Call {
  int mode = FWD;
  Prob a{};           // geometry, GEMM extents, class fields, output, beta
  const void* A = nullptr;  // operand base pointers (x / dy / w)
  const void* B = nullptr;
  int key[14] = {};   // autotune key
};
struct Cfg {
  int bn = 0, splits = 0;
  int cm = 1;  // CTAs per cluster sharing the B tile by multicast (1 or 2; FWD / DGRAD)
  int bs = 0;  // B-stationary (FWD / DGRAD, splits 1, cm 1, B tile <= kMaxBStat bytes)
  int sk = 0;  // stream-K over all CTA slots with the in-kernel fix-up (cm 1, bs 0)
};
constexpr size_t kMaxBStat = 128 * 1024;
struct KeyHash {
  size_t operator()(const std::array<int, 14>& k) const {
    size_t h = 1469598103934665603ull;
    for (int v : k) h = (h ^ static_cast<size_t>(v)) * 1099511628211ull;
    return h;
  }
};
std::unordered_map<std::array<int, 14>, Cfg, KeyHash> g_tuned;
int g_autotune = 0;

bool bn_ok(const Call& c, int bn) {
  switch (c.mode) {
    case FWD:
      return bn == 64 || c.a.K > bn / 2;  // no tile wider than twice the channels
    case DGRAD:
      return (c.a.C % bn == 0 || bn == 64) && (bn == 64 || c.a.C > bn / 2);
    default:
      return c.a.C % bn == 0;
  }
}

bool encode(const Call& c, int bn, int cm, CUtensorMap* ta, CUtensorMap* tb, Prob& a) {
  if (c.mode == FWD) {
    bool ok;
    if (a.a_tiled) {
      const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.C), static_cast<cuuint64_t>(a.M)};
      const cuuint64_t str[1] = {static_cast<cuuint64_t>(a.C) * 4};
      const cuuint32_t box[2] = {32, kBM};
      ok = tiled_map(ta, c.A, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
      const int lo = -a.pad, up = a.pad - (a.R - 1);
      ok = im2col_map(ta, c.A, a.N, a.H, a.W, a.C, lo, lo, up, up, a.stride, kBM,
                      CU_TENSOR_MAP_SWIZZLE_128B);
    }
    const int Kg = a.R * a.S * a.C;
    const cuuint64_t bd[2] = {static_cast<cuuint64_t>(Kg), static_cast<cuuint64_t>(a.K)};
    const cuuint64_t bs[1] = {static_cast<cuuint64_t>(Kg) * 4};
    const cuuint32_t bbox[2] = {32, static_cast<cuuint32_t>(bn / cm)};  // cm: half per CTA
    return ok && tiled_map(tb, c.B, 2, bd, bs, bbox, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (c.mode == DGRAD) {
    bool ok;
    if (a.a_tiled) {
      const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.K),
                                  static_cast<cuuint64_t>(a.N) * a.P * a.Q};
      const cuuint64_t str[1] = {static_cast<cuuint64_t>(a.K) * 4};
      const cuuint32_t box[2] = {32, kBM};
      ok = tiled_map(ta, c.A, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
      ok = im2col_map(ta, c.A, a.N, a.P, a.Q, a.K, a.lo_h, a.lo_w, a.Hc - a.P + a.lo_h,
                      a.Wc - a.Q + a.lo_w, 1, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    if (!ok) return false;
    // B: all BN/32 MN atoms (32 ci x 32 co) of a stage as one 4-D box over
    // w viewed as {ci 32, co, ci-block, tap}; else one 3-D box per atom
    a.b_packed = 0;
    if (a.C % 32 == 0 && a.C >= bn) {
      const cuuint64_t pd[4] = {32, static_cast<cuuint64_t>(a.K), static_cast<cuuint64_t>(a.C / 32),
                                static_cast<cuuint64_t>(a.R) * a.S};
      const cuuint64_t ps[3] = {static_cast<cuuint64_t>(a.C) * a.R * a.S * 4, 128,
                                static_cast<cuuint64_t>(a.C) * 4};
      const cuuint32_t pbox[4] = {32, 32, static_cast<cuuint32_t>(bn / 32 / cm), 1};
      if (tiled_map(tb, c.B, 4, pd, ps, pbox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
        a.b_packed = 1;
        return true;
      }
    }
    const cuuint64_t bd[3] = {static_cast<cuuint64_t>(a.C), static_cast<cuuint64_t>(a.R) * a.S,
                              static_cast<cuuint64_t>(a.K)};
    const cuuint64_t bs[2] = {static_cast<cuuint64_t>(a.C) * 4,
                              static_cast<cuuint64_t>(a.C) * a.R * a.S * 4};
    const cuuint32_t bbox[3] = {32, 1, 32};
    return tiled_map(tb, c.B, 3, bd, bs, bbox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  }
  const int Kg = a.N * a.P * a.Q;
  // A: dy as {co 32, pixel, co-block} (4 atoms per box) when Cout % 32 == 0
  a.a_packed = 0;
  bool ok = false;
  if (a.K % 32 == 0) {
    const cuuint64_t pd[3] = {32, static_cast<cuuint64_t>(Kg), static_cast<cuuint64_t>(a.K / 32)};
    const cuuint64_t ps[2] = {static_cast<cuuint64_t>(a.K) * 4, 128};
    const cuuint32_t pbox[3] = {32, 32, kBM / 32};
    ok = tiled_map(ta, c.A, 3, pd, ps, pbox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    a.a_packed = ok ? 1 : 0;
  }
  if (!ok) {
    const cuuint64_t ad[2] = {static_cast<cuuint64_t>(a.K), static_cast<cuuint64_t>(Kg)};
    const cuuint64_t as[1] = {static_cast<cuuint64_t>(a.K) * 4};
    const cuuint32_t abox[2] = {32, 32};
    if (!tiled_map(ta, c.A, 2, ad, as, abox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return false;
  }
  // B: 1x1 stride-1 unpadded convs read x as a plain {ci 32, pixel, ci-block} box
  a.b_packed = 0;
  if (a.R == 1 && a.S == 1 && a.stride == 1 && a.pad == 0) {
    const cuuint64_t pd[3] = {32, static_cast<cuuint64_t>(Kg), static_cast<cuuint64_t>(a.C / 32)};
    const cuuint64_t ps[2] = {static_cast<cuuint64_t>(a.C) * 4, 128};
    const cuuint32_t pbox[3] = {32, 32, static_cast<cuuint32_t>(bn / 32)};
    if (tiled_map(tb, c.B, 3, pd, ps, pbox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
      a.b_packed = 1;
      return true;
    }
  }
  const int lo = -a.pad, up = a.pad - (a.R - 1);
  return im2col_map(tb, c.B, a.N, a.H, a.W, a.C, lo, lo, up, up, a.stride, 32,
                    CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

template <int MODE, int CM, int BS, int G = 1>
int dispatch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const Prob& a,
                int bn, cudaStream_t st) {
  if constexpr (CM == 1 && BS == 0 && G == 1) {
    if (a.streamk) {
      if (bn == 256) return launch_t<MODE, 256, 4, 1, 0, 1, 1>(ta, tb, tc, a, st);
      if (bn == 128) return launch_t<MODE, 128, 6, 1, 0, 1, 1>(ta, tb, tc, a, st);
      return launch_t<MODE, 64, 8, 1, 0, 1, 1>(ta, tb, tc, a, st);
    }
  }
  if (BS) {  // A-only ring of 4 x 16 KB; B lives in its own region
    if (bn == 256) return launch_t<MODE, 256, 4, CM, BS, 1>(ta, tb, tc, a, st);
    if (bn == 128) return launch_t<MODE, 128, 4, CM, BS, 1>(ta, tb, tc, a, st);
    return launch_t<MODE, 64, 4, CM, BS, 1>(ta, tb, tc, a, st);
  }
  if (G == 2) {  // 32 / 24 / 20 KB stages
    if (bn == 256) return launch_t<MODE, 256, 6, CM, BS, G>(ta, tb, tc, a, st);
    if (bn == 128) return launch_t<MODE, 128, 8, CM, BS, G>(ta, tb, tc, a, st);
    return launch_t<MODE, 64, 8, CM, BS, G>(ta, tb, tc, a, st);
  }
  if (bn == 256) return launch_t<MODE, 256, 4, CM, BS, 1>(ta, tb, tc, a, st);
  if (bn == 128) return launch_t<MODE, 128, 6, CM, BS, 1>(ta, tb, tc, a, st);
  return launch_t<MODE, 64, 8, CM, BS, 1>(ta, tb, tc, a, st);
}

template <int MODE>
int dispatch_kc(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const Prob& a,
                int bn, cudaStream_t st) {
  // one ring stage fewer than the plain kernels: the receive slots take 32 KB
  if (bn == 256) return launch_t<MODE, 256, 3, 1, 0, 1, 0, 1>(ta, tb, tc, a, st);
  if (bn == 128) return launch_t<MODE, 128, 5, 1, 0, 1, 0, 1>(ta, tb, tc, a, st);
  return launch_t<MODE, 64, 6, 1, 0, 1, 0, 1>(ta, tb, tc, a, st);
}

// -1: could not encode the tensor maps (not launched)
int launch_cfg(const Call& c, Cfg cfg, cudaStream_t st) {
  CUtensorMap ta, tb;
  Prob a = c.a;
  // cm 5: split-K over a CTA pair, reduced through DSMEM (FWD / DGRAD,
  // row-major outputs written by the bulk-store epilogue, 2 slices)
  const bool kc = cfg.cm == 5;
  if (kc) {
    if (c.mode == WGRAD || cfg.splits != 2 || cfg.bs || cfg.sk || a.scatter || a.stats) return -1;
    cfg.cm = 1;
  }
  // cm 6: 2-slice split-K reduced by bulk reduce-adds into the zeroed output
  // (overwrite calls with row-major outputs only: with beta = 1 the old value
  // would make the order matter); cm 7 / 8: the same over 2-SM MMA pairs
  // (cm 2 / cm 4 tiles, each CTA of the pair reduce-adds its own 128 rows)
  const bool padd = cfg.cm >= 6;
  if (padd) {
    if (cfg.splits != 2 || cfg.bs || cfg.sk || a.scatter || a.stats || a.beta) return -1;
    if (a.kb_total < 2) return -1;  // both slices must own k-blocks
    if (cfg.cm > 6 && c.mode == WGRAD) return -1;
    cfg.cm = cfg.cm == 6 ? 1 : cfg.cm == 7 ? 2 : 4;
  }
  if (c.mode == WGRAD) cfg.cm = 1;  // multicast of B across M-tiles: FWD / DGRAD only
  if (cfg.bs && (c.mode == WGRAD || cfg.splits != 1 || cfg.cm != 1 ||
                 static_cast<size_t>(c.a.kb_total) * cfg.bn * kBK * 4 > kMaxBStat))
    cfg.bs = 0;
  // cm 4: CTA pair running 2-SM MMAs (each CTA loads half of the B columns, like cm 2)
  if (!encode(c, cfg.bn, cfg.cm > 1 ? 2 : 1, &ta, &tb, a)) return -1;
  a.tiles_m = (a.M + kBM - 1) / kBM;
  a.tiles_n = (a.Ng + cfg.bn - 1) / cfg.bn;
  a.splits = cfg.splits;
  a.ws = g_cur->ws;
  a.trace = g_trace;
  a.streamk = 0;
  if (cfg.sk) {
    // stream-K: G CTAs share the tile-major (tile, k-block) iterations
    if (cfg.cm != 1 || cfg.bs || a.stats) return -1;
    const long long tiles = static_cast<long long>(a.tiles_m) * a.tiles_n;
    const long long T = tiles * a.kb_total;
    const int G = static_cast<int>(std::min<long long>(T, cta_slots()));
    if (tiles > kMaxFixTiles || G < 1) return -1;
    int maxseg = 1;
    for (long long t = 0; t < tiles; ++t)
      maxseg = std::max(maxseg, sk_cta_of(t * a.kb_total + a.kb_total - 1, T, G) -
                                    sk_cta_of(t * a.kb_total, T, G) + 1);
    if (maxseg > 1 && (static_cast<size_t>(tiles) * maxseg * kBM * cfg.bn * 4 > ws_capacity() ||
                       !fix_counters(*g_cur)))
      return -1;
    a.streamk = 1;
    a.sk_maxseg = maxseg;
    a.fix_cnt = fix_counters(*g_cur);
    a.splits = 1;
    a.kb_per_split = a.kb_total;
    a.units = static_cast<int>(std::min<long long>(T, 1 << 30));  // grid = min(T, CTA slots)
  } else if (kc) {
    a.kb_per_split = (a.kb_total + 1) / 2;
    if (a.kb_per_split >= a.kb_total) return -1;  // one k-block: nothing to split
    a.units = a.tiles_m * a.tiles_n;  // per CTA pair
  } else {
    a.kb_per_split = (a.kb_total + a.splits - 1) / a.splits;
    a.units = (cfg.cm > 1 ? (a.tiles_m + 1) / 2 : a.tiles_m) * a.tiles_n * a.splits;
  }
  // output tensor map for the bulk-store epilogue: the split-K workspace
  // {Ng, M, S} (rows past M clip inside their own slice) or the row-major
  // output {Ng, M}; scatter outputs (strided dgrad classes) store directly
  CUtensorMap tc;
  std::memset(&tc, 0, sizeof(tc));
  a.tma_out = 0;
  a.pair_add = padd ? 1 : 0;
  if (a.splits > 1 && !kc && !padd) {
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.Ng), static_cast<cuuint64_t>(a.M),
                                static_cast<cuuint64_t>(a.splits)};
    const cuuint64_t str[2] = {static_cast<cuuint64_t>(a.Ng) * 4,
                               static_cast<cuuint64_t>(a.Ng) * a.M * 4};
    const cuuint32_t box[3] = {32, 32, 1};
    a.tma_out = tiled_map(&tc, a.ws, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B) ? 1 : 0;
  } else if (!a.scatter) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.Ng), static_cast<cuuint64_t>(a.M)};
    const cuuint64_t str[1] = {static_cast<cuuint64_t>(a.Ng) * 4};
    const cuuint32_t box[2] = {32, 32};
    a.tma_out = tiled_map(&tc, a.out, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B) ? 1 : 0;
  }
  if (cfg.bs && a.tiles_n > sm_count()) cfg.bs = 0;
  if (padd) {
    if (!a.tma_out) return -1;
    const cudaError_t e =
        cudaMemsetAsync(a.out, 0, sizeof(float) * static_cast<size_t>(a.M) * a.Ng, st);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  if (kc) {
    if (!a.tma_out) return -1;
    return c.mode == FWD ? dispatch_kc<FWD>(ta, tb, tc, a, cfg.bn, st)
                         : dispatch_kc<DGRAD>(ta, tb, tc, a, cfg.bn, st);
  }
  if (c.mode == FWD)
    return cfg.bs ? dispatch_bn<FWD, 1, 1>(ta, tb, tc, a, cfg.bn, st)
           : cfg.cm == 4 ? dispatch_bn<FWD, 2, 0, 2>(ta, tb, tc, a, cfg.bn, st)
           : cfg.cm > 1  ? dispatch_bn<FWD, 2, 0>(ta, tb, tc, a, cfg.bn, st)
                         : dispatch_bn<FWD, 1, 0>(ta, tb, tc, a, cfg.bn, st);
  if (c.mode == DGRAD)
    return cfg.bs ? dispatch_bn<DGRAD, 1, 1>(ta, tb, tc, a, cfg.bn, st)
           : cfg.cm == 4 ? dispatch_bn<DGRAD, 2, 0, 2>(ta, tb, tc, a, cfg.bn, st)
           : cfg.cm > 1  ? dispatch_bn<DGRAD, 2, 0>(ta, tb, tc, a, cfg.bn, st)
                         : dispatch_bn<DGRAD, 1, 0>(ta, tb, tc, a, cfg.bn, st);
  return dispatch_bn<WGRAD, 1, 0>(ta, tb, tc, a, cfg.bn, st);
}

bool splits_ok(const Call& c, int s) {
  if (s < 1 || s > c.a.kb_total) return false;
  const int per = (c.a.kb_total + s - 1) / s;
  if ((c.a.kb_total + per - 1) / per != s) return false;
  return s == 1 || static_cast<size_t>(s) * c.a.M * c.a.Ng * 4 <= ws_capacity();
}

Cfg model_cfg(const Call& c) {
  int bn;
  if (c.mode == FWD) bn = c.a.K >= 256 ? 256 : (c.a.K > 64 ? 128 : 64);
  else if (c.mode == DGRAD) bn = c.a.C >= 256 ? 256 : (c.a.C > 64 ? 128 : 64);
  else bn = (c.a.C % 256 == 0) ? 256 : (c.a.C % 128 == 0) ? 128 : 64;
  if (!bn_ok(c, bn)) bn = 64;
  const long long tiles =
      static_cast<long long>((c.a.M + kBM - 1) / kBM) * ((c.a.Ng + bn - 1) / bn);
  Cfg cfg;
  cfg.bn = bn;
  cfg.splits = choose_splits(tiles, c.a.kb_total, bn, static_cast<long long>(c.a.M) * c.a.Ng,
                             c.a.beta, ws_capacity());
  return cfg;
}

// Empirical choice of (BN, splits) for one GEMM: every candidate is run
// once and then timed (min of 3, CUDA events on the caller's stream), never
// during stream capture; accumulating (beta = 1) calls are tuned on a scratch
// output.  The result is cached per shape for the life of the process.
// Seconds per launch of a candidate as the captured step runs it: a CUDA graph
// of kTuneReps back-to-back launches on the tuning stream, best of two
// replays.  (Timed eagerly, the host launch gaps and the pair-add memset's
// own launch would be charged to every candidate; the step pays neither.)
constexpr int kTuneReps = 4;
bool tune_eager() {  // ACCUDNN_TUNE_EAGER=1: time candidates as eager single launches
  static const bool v = [] {
    const char* e = std::getenv("ACCUDNN_TUNE_EAGER");
    return e && std::atoi(e) != 0;
  }();
  return v;
}
float time_in_graph(const Call& c, const Cfg& cand, cudaStream_t ts, cudaEvent_t e0,
                    cudaEvent_t e1) {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  if (cudaStreamBeginCapture(ts, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return 1e30f;
  }
  bool ok = true;
  for (int i = 0; i < kTuneReps && ok; ++i) ok = launch_cfg(c, cand, ts) == 0;
  const cudaError_t ec = cudaStreamEndCapture(ts, &g);
  float best = 1e30f;
  if (ok && ec == cudaSuccess && g && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess) {
    cudaGraphLaunch(ge, ts);  // warm: tensor maps, L2
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0, ts);
      cudaGraphLaunch(ge, ts);
      cudaEventRecord(e1, ts);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms / kTuneReps);
    }
  }
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
  return best;
}

Cfg tune(const Call& c, cudaStream_t st) {
  static const int kSplits[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 48, 64, 96, 128};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // candidates run on a private stream ordered after the caller's work (the
  // caller's stream may be the legacy stream, which cannot be captured); the
  // caller's stream waits for them at the end (same workspace)
  static cudaStream_t ts = [] {
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    return s;
  }();
  cudaEvent_t dep;
  cudaEventCreateWithFlags(&dep, cudaEventDisableTiming);
  cudaEventRecord(dep, st);
  cudaStreamWaitEvent(ts, dep, 0);
  Cfg best = model_cfg(c);
  float best_ms = 1e30f;
  // 0: plain, 1: 2-CTA multicast, 3: 2-SM MMA pair.  (2, B-stationary, is
  // available through accudnn_conv_force_cfg but not tuned: measured no faster)
  // 5: split-K over a DSMEM-reduced CTA pair (2 slices); 6 / 7 / 8: 2 slices reduce-added
  // into the zeroed output by single CTAs / 2-SM pairs / multicast pairs
  static const int max_variant = [] {  // ACCUDNN_TUNE_VARIANTS: highest variant tried
    const char* e = std::getenv("ACCUDNN_TUNE_VARIANTS");
    return e ? std::atoi(e) : 8;
  }();
  for (int variant : {0, 1, 3, 5, 6, 7, 8}) {
   if (variant > max_variant) continue;
   const int cm = variant == 1 ? 2 : variant == 3 ? 4 : variant >= 5 ? variant : 1;
   const int bs = variant == 2 ? 1 : 0;
   if (variant > 0 && c.mode == WGRAD) continue;
   for (int bn : {64, 128, 256}) {
    if (!bn_ok(c, bn)) continue;
    if (bs && static_cast<size_t>(c.a.kb_total) * bn * kBK * 4 > kMaxBStat) continue;
    for (int s : kSplits) {
     // s = 0: stream-K (single-CTA tiles only)
     for (int sk : {0, 1}) {
      if (sk && (s != 1 || cm != 1 || bs)) continue;
      if (cm >= 5 && (s != 2 || sk)) continue;
      if (!splits_ok(c, s)) continue;
      if (bs && s != 1) continue;
      const Cfg cand{bn, s, cm, bs, sk};
      if (launch_cfg(c, cand, ts) != 0) {
        cudaGetLastError();
        continue;
      }
      float t = 1e30f;
      if (tune_eager()) {  // A/B: eager single launches (the round-1 tuner)
        for (int r = 0; r < 3; ++r) {
          cudaEventRecord(e0, ts);
          launch_cfg(c, cand, ts);
          cudaEventRecord(e1, ts);
          cudaEventSynchronize(e1);
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          t = std::min(t, ms);
        }
      } else {
        t = time_in_graph(c, cand, ts, e0, e1);
      }
      if (t < best_ms) {
        best_ms = t;
        best = cand;
      }
     }
    }
   }
  }
  cudaEventRecord(dep, ts);
  cudaStreamWaitEvent(st, dep, 0);
  cudaEventDestroy(dep);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

Cfg g_force{0, 0, 0};  // test hook (accudnn_conv_force_cfg): fields > 0 override

int run_call(const Call& c, cudaStream_t st) {
  static const bool drain_set = [] {
    const char* e = std::getenv("ACCUDNN_CONV_DRAIN");
    const int v = e ? std::atoi(e) : 0;
    if (v) cudaMemcpyToSymbol(g_conv_drain, &v, sizeof(v));
    return true;
  }();
  (void)drain_set;
  if (g_force.bn > 0 || g_force.splits != 0 || g_force.cm > 0) {
    Cfg f = model_cfg(c);
    if (g_force.bn > 0 && bn_ok(c, g_force.bn)) f.bn = g_force.bn;
    if (g_force.splits > 0 && splits_ok(c, g_force.splits)) f.splits = g_force.splits;
    if (g_force.splits == -1) {  // stream-K; falls back where not eligible
      Cfg k = f;
      k.splits = 1;
      k.cm = 1;
      k.sk = 1;
      const int r = launch_cfg(c, k, st);
      if (r != -1) return r;
    }
    if (g_force.cm > 0) f.cm = g_force.cm == 3 ? 1 : g_force.cm;
    if (g_force.cm == 3) {  // test hook: B-stationary
      f.bs = 1;
      f.splits = 1;
    }
    if (g_force.cm >= 6) {  // test hook: 2-slice split-K by reduce-adds into the zeroed output
      f.splits = 2;
      f.bs = 0;
      f.sk = 0;
      const int r = launch_cfg(c, f, st);
      if (r != -1) return r;
      f = model_cfg(c);
    }
    if (g_force.cm == 5) {  // test hook: split-K pair reduced through DSMEM
      f.splits = 2;
      f.bs = 0;
      f.sk = 0;
      const int r = launch_cfg(c, f, st);
      if (r != -1) return r;
      f = model_cfg(c);  // not eligible (WGRAD, scatter output, one k-block)
    }
    return launch_cfg(c, f, st);
  }
  std::array<int, 14> key;
  std::copy(std::begin(c.key), std::end(c.key), key.begin());
  Cfg cfg;
  auto it = g_tuned.find(key);
  // (the 2-slice pair schedules, cm 5 / 6, need no split-K workspace)
  if (it != g_tuned.end() &&
      (it->second.cm >= 5 ? c.a.kb_total >= 2 : splits_ok(c, it->second.splits))) {
    cfg = it->second;
  } else {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    if (g_autotune && cap == cudaStreamCaptureStatusNone) {
      if (!c.a.beta) {
        cfg = tune(c, st);
        g_tuned[key] = cfg;
      } else {
        // accumulating calls are tuned against a scratch copy of the output
        // (the candidates add into it; the real output is left untouched)
        const size_t out_bytes =
            sizeof(float) * (c.mode == DGRAD ? static_cast<size_t>(c.a.N) * c.a.H * c.a.W * c.a.C
                                             : static_cast<size_t>(c.a.M) * c.a.Ng);
        float* scratch = nullptr;
        if (cudaMalloc(&scratch, out_bytes) == cudaSuccess) {
          Call c2 = c;
          c2.a.out = scratch;
          cfg = tune(c2, st);
          cudaStreamSynchronize(st);
          cudaFree(scratch);
          g_tuned[key] = cfg;
        } else {
          cudaGetLastError();
          cfg = model_cfg(c);
        }
      }
    } else {
      cfg = model_cfg(c);
    }
  }
  int r = launch_cfg(c, cfg, st);
  // a tuned stream-K or K-split-pair entry that this call cannot use (a smaller
  // workspace now, BN statistics requested): the analytic config instead
  if (r == -1 && (cfg.sk || cfg.cm >= 5)) r = launch_cfg(c, model_cfg(c), st);
  return r;
}

void fill_key(Call& c, const accudnn_conv_desc* d, int cls) {
  const int k[14] = {c.mode, d->n, d->h, d->w, d->c, d->k, d->r, d->s, d->stride, d->pad,
                     d->p, d->q, cls, 0};
  std::copy(k, k + 14, c.key);
}

}  // namespace

// 0 = not eligible (caller falls back to the cp.async kernel), else launched
int conv_tma_fwd(const accudnn_conv_desc* d, const float* x, const float* w, float* y, int beta,
                 cudaStream_t st, int* rc, float* stats) {
  if (!geometry_ok(d) || (d->c % 32) || (d->k % 4)) return 0;
  Call c;
  c.mode = FWD;
  Prob& a = c.a;
  a = base_prob(d);
  a.M = a.N * a.P * a.Q;
  a.Ng = a.K;
  a.kb_total = a.R * a.S * a.C / kBK;
  a.out = y;
  a.beta = beta;
  a.stats = (beta || a.K % 32) ? nullptr : stats;
  a.a_tiled = (a.R == 1 && a.stride == 1 && a.pad == 0);
  c.A = x;
  c.B = w;
  fill_key(c, d, 0);
  const int r = run_call(c, st);
  if (r == -1) return 0;
  *rc = r;
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
  *rc = 0;
  bool launched = false;
  if (any_empty && !beta) {
    // zero only the pixels no class GEMM writes (the others are written, not
    // accumulated, by their class)
    unsigned row_empty = 0, col_empty = 0;
    for (int c = 0; c < s; ++c) {
      if (rows[c].taps == 0) row_empty |= 1u << c;
      if (cols[c].taps == 0) col_empty |= 1u << c;
    }
    const int grid = static_cast<int>(std::min<long long>(static_cast<long long>(d->n) * d->h,
                                                          16LL * sm_count()));
    launch_pdl(dgrad_zero_empty_kernel, grid, 256, 0, st, reinterpret_cast<float4*>(dx), d->n, d->h,
               d->w, d->c / 4, s, row_empty, col_empty);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      *rc = static_cast<int>(e);
      return 1;
    }
    launched = true;
  }
  for (int ca = 0; ca < s; ++ca) {
    for (int cb = 0; cb < s; ++cb) {
      const ClassDim& cr = rows[ca];
      const ClassDim& cc = cols[cb];
      if (cr.taps == 0 || cc.taps == 0) continue;
      Call c;
      c.mode = DGRAD;
      Prob& a = c.a;
      a = base_prob(d);
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
      c.A = dy;
      c.B = w;
      fill_key(c, d, 1 + ca * s + cb);
      c.key[13] = beta;
      const int r = run_call(c, st);
      if (r == -1) return launched ? (*rc = static_cast<int>(cudaErrorInvalidValue), 1) : 0;
      launched = true;
      *rc = r;
      if (r) return 1;
    }
  }
  return 1;
}

int conv_tma_wgrad(const accudnn_conv_desc* d, const float* x, const float* dy, float* dw,
                   int beta, cudaStream_t st, int* rc) {
  if (!geometry_ok(d) || (d->c % 32) || (d->k % 4) || (d->c % 64)) return 0;
  Call c;
  c.mode = WGRAD;
  Prob& a = c.a;
  a = base_prob(d);
  a.M = a.K;
  a.Ng = a.R * a.S * a.C;
  // a ragged last K-block reads past the last output pixel: the im2col walk
  // and the dy tile land out of bounds there and are zero-filled by the TMA
  a.kb_total = (a.N * a.P * a.Q + kBK - 1) / kBK;
  a.out = dw;
  a.beta = beta;
  c.A = dy;
  c.B = x;
  fill_key(c, d, 0);
  const int r = run_call(c, st);
  if (r == -1) return 0;
  *rc = r;
  return 1;
}

void conv_select_workspace(cudaStream_t st) {
  g_cur = &g_ws;
  g_cur_ctas = 0;
  for (const auto& e : g_stream_ws)
    if (e->st == st) {
      // a registered stream always uses its own workspace (none: no split-K),
      // never another stream's
      g_cur = &e->w;
      g_cur_ctas = e->max_ctas;
    }
}

// shared with the cp.async kernel (conv_igemm.cu): the split-K workspace if
// it holds `bytes`, else nullptr; and the slice-order reduction on it
float* conv_splitk_workspace(size_t bytes) {
  return ws_capacity() >= bytes ? g_cur->ws : nullptr;
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
  launch_pdl(conv_splitk_reduce_kernel, rgrid, 256, 0, st, a);
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
  zero_fix_counters(g_ws);
  return 0;
}

// a split-K workspace used only by convolutions launched on `stream` (an
// executor's compute stream, or its weight-gradient stream running
// concurrently with it) and a cap on their persistent grids (max_ctas SMs,
// 0 = all).  ptr == NULL, bytes == 0 and max_ctas == 0 removes the stream's
// entry; ptr == NULL with max_ctas < 0 registers the stream without a
// workspace (its convolutions never split K).
extern "C" int accudnn_conv_set_stream_workspace(void* stream, void* ptr,
                                                 unsigned long long bytes, int max_ctas) {
  using namespace accudnn;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!st) return static_cast<int>(cudaErrorInvalidValue);
  for (size_t i = 0; i < g_stream_ws.size(); ++i)
    if (g_stream_ws[i]->st == st) {
      if (g_cur == &g_stream_ws[i]->w) g_cur = &g_ws;
      g_stream_ws.erase(g_stream_ws.begin() + static_cast<long>(i));
      break;
    }
  if (!ptr && bytes == 0 && max_ctas == 0) return 0;
  auto e = std::make_unique<StreamWs>();
  e->st = st;
  e->w.ws = static_cast<float*>(ptr);
  e->w.bytes = ptr ? static_cast<size_t>(bytes) : 0;
  e->max_ctas = std::max(0, max_ctas);
  zero_fix_counters(e->w);
  g_stream_ws.push_back(std::move(e));
  return 0;
}

// debug: subsequent TMA-conv launches record clock64 stamps into buf
// (1024 int64 per CTA: [0,256) producer issue of k-block i, [256,512) MMA
// start of k-block i, [512,768) epilogue start/end of unit j); NULL = off
extern "C" int accudnn_conv_trace(void* buf) {
  accudnn::g_trace = static_cast<long long*>(buf);
  return 0;
}

// The tuned table as text, one entry per line:
// "k0 k1 ... k13 bn splits cm bs sk\n" (the 14-int shape key, see fill_key).  The
// returned buffer is malloc'ed; release it with free() (accudnn_rt_free).
extern "C" int accudnn_conv_tune_export(char** out) {
  std::string t;
  for (const auto& kv : accudnn::g_tuned) {
    for (int v : kv.first) t += std::to_string(v) + " ";
    t += std::to_string(kv.second.bn) + " " + std::to_string(kv.second.splits) + " " +
         std::to_string(kv.second.cm) + " " + std::to_string(kv.second.bs) + " " +
         std::to_string(kv.second.sk) + "\n";
  }
  char* buf = static_cast<char*>(std::malloc(t.size() + 1));
  if (!buf) return static_cast<int>(cudaErrorMemoryAllocation);
  std::memcpy(buf, t.c_str(), t.size() + 1);
  *out = buf;
  return 0;
}
// merges entries in the export format into the table (overwriting)
extern "C" int accudnn_conv_tune_import(const char* text) {
  if (!text) return static_cast<int>(cudaErrorInvalidValue);
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    std::istringstream ls(line);
    std::array<int, 14> key;
    accudnn::Cfg cfg;
    bool ok = true;
    for (int& v : key) ok = ok && static_cast<bool>(ls >> v);
    ok = ok && static_cast<bool>(ls >> cfg.bn >> cfg.splits);
    if (!ok) continue;
    if (!(ls >> cfg.cm) || (cfg.cm != 1 && cfg.cm != 2 && cfg.cm != 4 && (cfg.cm < 5 || cfg.cm > 8)))
      cfg.cm = 1;
    if (!(ls >> cfg.bs) || (cfg.bs != 0 && cfg.bs != 1)) cfg.bs = 0;
    if (!(ls >> cfg.sk) || (cfg.sk != 0 && cfg.sk != 1)) cfg.sk = 0;
    if (cfg.bn != 64 && cfg.bn != 128 && cfg.bn != 256) continue;
    if (cfg.splits < 1) continue;
    accudnn::g_tuned[key] = cfg;
  }
  return 0;
}

// test hook: force (tile width, split-K factor, cluster size) for every TMA
// conv launch (0 = automatic; an invalid width or split falls back)
extern "C" int accudnn_conv_force_cfg(int bn, int splits, int cm) {
  accudnn::g_force = accudnn::Cfg{bn, splits, cm};
  return 0;
}

// 1: tune (BN, split-K) per convolution shape on first use (beta = 0 calls,
// outside stream capture), 0: analytic choice.  Returns the previous mode.
extern "C" int accudnn_conv_autotune(int enable) {
  const int prev = accudnn::g_autotune;
  accudnn::g_autotune = enable ? 1 : 0;
  return prev;
}
