// SM-driven featuremap transfers between the device arena and pinned host
// memory (the swap executor's alternative to copy-engine cudaMemcpyAsync).
//
// The reference's runtime model charges a transfer bytes / bandwidth
// (perf_model.cpp:112-132, simulator.cpp:233-285): no per-copy cost.  A
// copy-engine memcpy pays ~3 us of issue/completion latency per call on
// B200 (measured: a 512 KB D2H takes 11.7 us + a 2-3 us gap to the next one
// in a CUDA graph, 38 GB/s effective; 128 KB runs at 15 GB/s), so a swap
// plan of many small featuremaps runs far below the link rate the model
// assumes.  This kernel moves the bytes with loads/stores through the
// host-mapped pinned buffer (UVA): D2H stores are posted writes over the
// link, H2D loads keep `kInFlight` 16-byte requests per thread outstanding
// to cover the link's round-trip latency.  A handful of CTAs saturate the
// link while the compute kernels keep the rest of the SMs.
#include <cuda_runtime.h>

#include <cstdint>

namespace accudnn {
namespace {

constexpr int kCopyThreads = 256;
constexpr int kInFlight = 8;

__global__ void __launch_bounds__(kCopyThreads) swap_copy_kernel(const uint4* __restrict__ src,
                                                                 uint4* __restrict__ dst,
                                                                 long long n16) {
  const long long stride = static_cast<long long>(gridDim.x) * kCopyThreads;
  // every batch keeps up to kInFlight loads outstanding, including the
  // ragged last one (a 128 KB transfer is a single batch: one link round
  // trip instead of one per 16-byte row of the grid)
  for (long long i = static_cast<long long>(blockIdx.x) * kCopyThreads + threadIdx.x; i < n16;
       i += kInFlight * stride) {
    uint4 v[kInFlight];
#pragma unroll
    for (int u = 0; u < kInFlight; ++u)
      if (i + u * stride < n16) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < kInFlight; ++u)
      if (i + u * stride < n16) __stcs(dst + i + u * stride, v[u]);
  }
}

__global__ void swap_copy_tail_kernel(const unsigned char* __restrict__ src,
                                      unsigned char* __restrict__ dst, int n) {
  if (threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
}

}  // namespace
}  // namespace accudnn

// bytes in any alignment; the 16-byte body by the vector kernel, the tail
// (< 16 B) by a one-warp kernel.  ctas <= 0: 16.
extern "C" int accudnn_swap_copy(void* dst, const void* src, unsigned long long bytes, int ctas,
                                 void* stream) {
  using namespace accudnn;
  if (!bytes) return 0;
  if (!dst || !src) return static_cast<int>(cudaErrorInvalidValue);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(src) % 16 == 0);
  const unsigned long long body = aligned ? bytes / 16 * 16 : 0;
  if (body) {
    const long long n16 = static_cast<long long>(body / 16);
    long long want = (n16 + kCopyThreads * kInFlight - 1) / (kCopyThreads * kInFlight);
    const int grid = static_cast<int>(want < 1 ? 1 : (want > (ctas > 0 ? ctas : 16) ? (ctas > 0 ? ctas : 16) : want));
    swap_copy_kernel<<<grid, kCopyThreads, 0, st>>>(static_cast<const uint4*>(src),
                                                    static_cast<uint4*>(dst), n16);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  unsigned long long rest = bytes - body;
  const unsigned char* s = static_cast<const unsigned char*>(src) + body;
  unsigned char* d = static_cast<unsigned char*>(dst) + body;
  while (rest) {
    const int n = static_cast<int>(rest > 1024 ? 1024 : rest);
    swap_copy_tail_kernel<<<1, 1024, 0, st>>>(s, d, n);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return static_cast<int>(e);
    rest -= static_cast<unsigned long long>(n);
    s += n;
    d += n;
  }
  return 0;
}
