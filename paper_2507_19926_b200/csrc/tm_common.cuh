// tm_common.cuh -- shared helpers of the sm_100a median kernels.
//
// Lane model.  Every median kernel works on 32-bit "lane words":
//   * 8- and 16-bit images: two independent problems packed as u16x2 -- the
//     low half-word belongs to lane 0, the high half-word to lane 1.  min/max
//     compile to VIMNMX.U16x2 / VIMNMX3.U16x2 (native on sm_100a, one
//     instruction for two selections);
//   * 32-bit images: one problem per word, VIMNMX.U32 / VIMNMX3.U32.
// 8-bit data is widened to 16-bit lanes (sm_100a has no native u8x4 min/max:
// __vminu4 lowers to LOP3/PRMT sequences -- profiles/r01_minmax_microbench.txt).
#pragma once
#include <atomic>
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace tmb {

template <typename T>
struct Lanes;

template <>
struct Lanes<uint8_t> {
  static constexpr int kLanes = 2;
  __device__ __forceinline__ static uint32_t mn(uint32_t a, uint32_t b) { return __vminu2(a, b); }
  __device__ __forceinline__ static uint32_t mx(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }
  __device__ __forceinline__ static uint32_t pack(uint8_t lo, uint8_t hi) {
    return (uint32_t)lo | ((uint32_t)hi << 16);
  }
  __device__ __forceinline__ static uint8_t lane(uint32_t w, int l) {
    return (uint8_t)(l ? (w >> 16) : (w & 0xFFFFu));
  }
};

template <>
struct Lanes<uint16_t> {
  static constexpr int kLanes = 2;
  __device__ __forceinline__ static uint32_t mn(uint32_t a, uint32_t b) { return __vminu2(a, b); }
  __device__ __forceinline__ static uint32_t mx(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }
  __device__ __forceinline__ static uint32_t pack(uint16_t lo, uint16_t hi) {
    return (uint32_t)lo | ((uint32_t)hi << 16);
  }
  __device__ __forceinline__ static uint16_t lane(uint32_t w, int l) {
    return (uint16_t)(l ? (w >> 16) : (w & 0xFFFFu));
  }
};

template <>
struct Lanes<uint32_t> {
  static constexpr int kLanes = 1;
  __device__ __forceinline__ static uint32_t mn(uint32_t a, uint32_t b) { return min(a, b); }
  __device__ __forceinline__ static uint32_t mx(uint32_t a, uint32_t b) { return max(a, b); }
  __device__ __forceinline__ static uint32_t pack(uint32_t lo, uint32_t) { return lo; }
  __device__ __forceinline__ static uint32_t lane(uint32_t w, int) { return w; }
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Shared-memory row padding: one extra word per 32 so that threads reading
// with a stride of 2, 4 or 8 words hit distinct banks (x + x/32 swizzle).
__host__ __device__ constexpr int padded(int x) { return x + (x >> 5); }

// Launch descriptor shared by all kernels: an image (or a band of one) with
// pitches in elements.  Rows [out_y0, out_y0 + out_h) of the source are
// filtered into dst rows [0, out_h); reads clamp to source rows [0, src_h)
// and columns [0, width), which are the *global* image edges -- a band with
// halo rows simply passes the halo as part of the source.
//
// Interleaved planes (H, W, C): `channels` > 1 makes blockIdx.z the channel;
// element (y, x) of channel c sits at base + y*pitch + x*channels + c.
struct Job {
  const void* src;
  void* dst;
  int64_t src_pitch;  // elements between rows
  int64_t dst_pitch;  // elements between rows
  int width;
  int src_h;
  int out_y0;
  int out_h;
  int channels;       // x stride in elements; 1 for a plain 2-D image
};

template <typename T>
__device__ __forceinline__ T load_px(const Job& job, int y, int x) {
  const T* s = static_cast<const T*>(job.src) + blockIdx.z;
  return __ldg(s + (int64_t)y * job.src_pitch + (int64_t)x * job.channels);
}

template <typename T>
__device__ __forceinline__ void store_px(const Job& job, int y, int x, T v) {
  T* d = static_cast<T*>(job.dst) + blockIdx.z;
  d[(int64_t)y * job.dst_pitch + (int64_t)x * job.channels] = v;
}

// Store N consecutive pixels of one row starting at x0 (masked at the right
// edge).  Plain 2-D destinations whose row segment is suitably aligned get one
// vector store instead of N scalar ones.
template <typename T, int N>
__device__ __forceinline__ void store_row(const Job& job, int y, int x0, const T (&v)[N]) {
  constexpr int kBytes = N * (int)sizeof(T);
  if (job.channels == 1 && x0 + N <= job.width && (kBytes == 4 || kBytes == 8 || kBytes == 16)) {
    T* d = static_cast<T*>(job.dst) + (int64_t)y * job.dst_pitch + x0;
    if ((reinterpret_cast<uintptr_t>(d) & (kBytes - 1)) == 0) {
      if constexpr (kBytes == 4) {
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < N; i++) w |= (uint32_t)v[i] << (8 * sizeof(T) * i);
        *reinterpret_cast<uint32_t*>(d) = w;
        return;
      } else if constexpr (kBytes == 8) {
        uint64_t w = 0;
#pragma unroll
        for (int i = 0; i < N; i++) w |= (uint64_t)v[i] << (8 * sizeof(T) * i);
        *reinterpret_cast<uint64_t*>(d) = w;
        return;
      } else if constexpr (kBytes == 16) {
        uint32_t w[4] = {0, 0, 0, 0};
        constexpr int per = 4 / (int)sizeof(T) > 0 ? 4 / (int)sizeof(T) : 1;
#pragma unroll
        for (int i = 0; i < N; i++) w[i / per] |= (uint32_t)v[i] << (8 * sizeof(T) * (i % per));
        *reinterpret_cast<uint4*>(d) = make_uint4(w[0], w[1], w[2], w[3]);
        return;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < N; i++)
    if (x0 + i < job.width) store_px<T>(job, y, x0 + i, v[i]);
}

// Per-kernel launch facts: opt-in shared-memory limit, SM count, resident CTAs
// per SM.  The shared-memory attribute is per device context, so the facts are
// kept per device ordinal (LaunchCache); a failed query is not cached.
struct LaunchInfo {
  cudaError_t err;
  int sms;
  int occ;
};
template <typename F>
inline LaunchInfo launch_info(F fn, int threads, int smem) {
  LaunchInfo li{cudaSuccess, 0, 1};
  li.err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (li.err != cudaSuccess) return li;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
  int o = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, smem);
  li.occ = o > 0 ? o : 1;
  return li;
}

// One per launcher (function-local static): launch facts per device ordinal,
// computed on the first launch on that device, thread-safe.
struct LaunchCache {
  static constexpr int kMaxDev = 64;
  std::atomic<int> ready[kMaxDev] = {};
  LaunchInfo info[kMaxDev] = {};
  std::mutex mu;
  template <typename F>
  LaunchInfo get(F fn, int threads, int smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev)
      return launch_info(fn, threads, smem);
    if (ready[dev].load(std::memory_order_acquire)) return info[dev];
    std::lock_guard<std::mutex> g(mu);
    if (!ready[dev].load(std::memory_order_relaxed)) {
      const LaunchInfo li = launch_info(fn, threads, smem);
      if (li.err != cudaSuccess) return li;  // not cached: a later call retries
      info[dev] = li;
      ready[dev].store(1, std::memory_order_release);
    }
    return info[dev];
  }
};

}  // namespace tmb
