// tm_med3.cu -- exact 3x3 median (k = 3) at memory speed.
//
// The reference's k = 3 program (oblivious.py:124-237 with root 1: column
// sorts + core merge + leaf selection, W(3) = 26 min/max per sample) is the
// textbook "forgetful" 3x3 selection: sort every column of three, then the
// median of the nine samples is med3(max of the column minima, med3 of the
// column medians, min of the column maxima).  Sharing every column sort
// between the three horizontally adjacent outputs that use it, this costs
// 6 min/max per column + 10 per output (3-input VIMNMX3 forms, native on
// sm_100a for u32 and u16x2) -- about 14 lane-ops per sample instead of 26.
//
// Layout: one thread = TX = 8 adjacent output columns x R output rows, for two
// row strips at once on u16x2 lanes (8/16-bit data; one strip for 32-bit).
// Three source rows live in registers and slide down one row per output row
// (each source row is loaded once per strip, +2 halo rows per strip); the
// loads are one vector per row (8 x T) plus two halo scalars, L1-shared with
// the neighbouring threads; clamped scalar loads only at the image edges or
// for unaligned / interleaved images.  Exact: pure min/max selection.
#include <cstdint>
#include <cuda_runtime.h>

#include "tm_common.cuh"
#include "tm_kernels.h"

namespace tmb {
namespace {

constexpr int TX = 8;
constexpr int NT = 128;

template <typename T>
struct M3;

template <>
struct M3<uint32_t> {
  static constexpr int L = 1;
  __device__ __forceinline__ static uint32_t mn(uint32_t a, uint32_t b) { return min(a, b); }
  __device__ __forceinline__ static uint32_t mx(uint32_t a, uint32_t b) { return max(a, b); }
  __device__ __forceinline__ static uint32_t mn3(uint32_t a, uint32_t b, uint32_t c) { return min(min(a, b), c); }
  __device__ __forceinline__ static uint32_t mx3(uint32_t a, uint32_t b, uint32_t c) { return max(max(a, b), c); }
};
struct M3u16x2 {
  static constexpr int L = 2;
  __device__ __forceinline__ static uint32_t mn(uint32_t a, uint32_t b) { return __vminu2(a, b); }
  __device__ __forceinline__ static uint32_t mx(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }
  __device__ __forceinline__ static uint32_t mn3(uint32_t a, uint32_t b, uint32_t c) { return __vminu2(__vminu2(a, b), c); }
  __device__ __forceinline__ static uint32_t mx3(uint32_t a, uint32_t b, uint32_t c) { return __vmaxu2(__vmaxu2(a, b), c); }
};
template <>
struct M3<uint16_t> : M3u16x2 {};
template <>
struct M3<uint8_t> : M3u16x2 {};

template <class M>
__device__ __forceinline__ uint32_t med3(uint32_t a, uint32_t b, uint32_t c) {
  return M::mx(M::mn(a, b), M::mn(M::mx(a, b), c));
}

// TX + 2 samples of one row (columns x0 - 1 .. x0 + TX), as 32-bit words.
template <typename T>
__device__ __forceinline__ void load_row(const T* rowp, int x0, int W, int CH, bool fast,
                                         uint32_t (&v)[TX + 2]) {
  if (fast) {  // x0 >= 1, x0 + TX < W, channels == 1, row + x0 aligned to 8 * sizeof(T)
    const T* p = rowp + x0;
    if constexpr (sizeof(T) == 1) {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
#pragma unroll
      for (int i = 0; i < 4; i++) {
        v[1 + i] = (w.x >> (8 * i)) & 0xFFu;
        v[5 + i] = (w.y >> (8 * i)) & 0xFFu;
      }
    } else if constexpr (sizeof(T) == 2) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(p));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; i++) {
        v[1 + 2 * i] = ws[i] & 0xFFFFu;
        v[2 + 2 * i] = ws[i] >> 16;
      }
    } else {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
      v[1] = a.x; v[2] = a.y; v[3] = a.z; v[4] = a.w;
      v[5] = b.x; v[6] = b.y; v[7] = b.z; v[8] = b.w;
    }
    v[0] = __ldg(p - 1);
    v[TX + 1] = __ldg(p + TX);
  } else {
#pragma unroll
    for (int i = 0; i < TX + 2; i++)
      v[i] = __ldg(rowp + (int64_t)clampi(x0 - 1 + i, 0, W - 1) * CH);
  }
}

template <typename T>
__global__ void __launch_bounds__(NT) med3_kernel(Job job, int R, int n_tx, int vec_ok) {
  using M = M3<T>;
  constexpr int L = M::L;
  const int chan = blockIdx.x % job.channels;
  const int xt = (blockIdx.x / job.channels) * NT + threadIdx.x;  // thread column tile
  if (xt >= n_tx) return;
  const int W = job.width, CH = job.channels;
  const int x0 = xt * TX;
  const T* src = static_cast<const T*>(job.src) + chan;
  T* dst = static_cast<T*>(job.dst) + chan;
  const int Yb = blockIdx.y * L * R;  // first output row (band-relative) of lane 0
  const bool fast = vec_ok && CH == 1 && x0 >= 1 && x0 + TX < W;

  // source row of strip s at sliding index q (output row t uses q = t, t+1, t+2)
  auto src_row = [&](int s, int q) {
    const int sy = clampi(job.out_y0 + Yb + s * R + q - 1, 0, job.src_h - 1);
    return src + (int64_t)sy * job.src_pitch;
  };
  // raw loads of sliding row q for both strips (issued one row ahead, packed
  // when consumed, so the load latency hides behind a row of compute)
  auto load_raw = [&](int q, uint32_t (&a)[TX + 2], uint32_t (&b)[TX + 2]) {
    load_row<T>(src_row(0, q), x0, W, CH, fast, a);
    if constexpr (L == 2) load_row<T>(src_row(1, q), x0, W, CH, fast, b);
  };
  auto pack = [&](const uint32_t (&a)[TX + 2], const uint32_t (&b)[TX + 2], uint32_t (&w)[TX + 2]) {
#pragma unroll
    for (int i = 0; i < TX + 2; i++) w[i] = L == 2 ? (a[i] | (b[i] << 16)) : a[i];
  };

  uint32_t r0[TX + 2], r1[TX + 2], r2[TX + 2];
  uint32_t na[TX + 2], nb[TX + 2];
  load_raw(0, na, nb);
  pack(na, nb, r0);
  load_raw(1, na, nb);
  pack(na, nb, r1);
  load_raw(2, na, nb);
  for (int t = 0; t < R; t++) {
    pack(na, nb, r2);
    if (t + 1 < R) load_raw(t + 3, na, nb);  // next row in flight during this row's compute
    uint32_t lo[TX + 2], md[TX + 2], hi[TX + 2];
#pragma unroll
    for (int c = 0; c < TX + 2; c++) {
      lo[c] = M::mn3(r0[c], r1[c], r2[c]);
      hi[c] = M::mx3(r0[c], r1[c], r2[c]);
      md[c] = med3<M>(r0[c], r1[c], r2[c]);
    }
    uint32_t o[TX];
#pragma unroll
    for (int i = 0; i < TX; i++) {
      const uint32_t a = M::mx3(lo[i], lo[i + 1], lo[i + 2]);
      const uint32_t b = med3<M>(md[i], md[i + 1], md[i + 2]);
      const uint32_t c = M::mn3(hi[i], hi[i + 1], hi[i + 2]);
      o[i] = med3<M>(a, b, c);
    }
#pragma unroll
    for (int s = 0; s < L; s++) {
      const int oy = Yb + s * R + t;
      if (oy < job.out_h) {
        T* d = dst + (int64_t)oy * job.dst_pitch;
        if (fast && vec_ok) {
          if constexpr (sizeof(T) == 1) {
            uint32_t w0 = 0, w1 = 0;
#pragma unroll
            for (int i = 0; i < 4; i++) {
              w0 |= ((o[i] >> (16 * s)) & 0xFFu) << (8 * i);
              w1 |= ((o[4 + i] >> (16 * s)) & 0xFFu) << (8 * i);
            }
            *reinterpret_cast<uint2*>(d + x0) = make_uint2(w0, w1);
          } else if constexpr (sizeof(T) == 2) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; i++)
              w[i] = ((o[2 * i] >> (16 * s)) & 0xFFFFu) | (((o[2 * i + 1] >> (16 * s)) & 0xFFFFu) << 16);
            *reinterpret_cast<uint4*>(d + x0) = make_uint4(w[0], w[1], w[2], w[3]);
          } else {
            *reinterpret_cast<uint4*>(d + x0) = make_uint4(o[0], o[1], o[2], o[3]);
            *(reinterpret_cast<uint4*>(d + x0) + 1) = make_uint4(o[4], o[5], o[6], o[7]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < TX; i++)
            if (x0 + i < W) d[(int64_t)(x0 + i) * CH] = (T)(L == 2 ? (o[i] >> (16 * s)) & 0xFFFFu : o[i]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < TX + 2; c++) {
      r0[c] = r1[c];
      r1[c] = r2[c];
    }
  }
}

template <typename T>
int launch_med3_t(const Job& job, cudaStream_t stream) {
  constexpr int L = M3<T>::L;
  static LaunchCache cache;
  const LaunchInfo li = cache.get(med3_kernel<T>, NT, 0);
  if (li.err != cudaSuccess) return (int)li.err;
  const int sms = li.sms;
  const int n_tx = (job.width + TX - 1) / TX;
  // rows per strip: enough threads for ~4 full waves of 2048 threads/SM, at
  // least 1 row (small images: parallelism over the 2 re-read halo rows)
  const long pair_rows = (job.out_h + L - 1) / L;
  const long want_threads = (long)sms * 2048 * 4;
  long R = (long)n_tx * job.channels * pair_rows / want_threads;
  R = R < 1 ? 1 : (R > 64 ? 64 : R);
  // short strips only when 4-row strips would fill less than a quarter wave
  if (R < 4 && 4 * (long)n_tx * job.channels * ((pair_rows + 3) / 4) >= (long)sms * 2048) R = 4;
  if (R > pair_rows) R = pair_rows;
  const uintptr_t base_s = reinterpret_cast<uintptr_t>(job.src);
  const uintptr_t base_d = reinterpret_cast<uintptr_t>(job.dst);
  const int vb = 8 * (int)sizeof(T) > 16 ? 16 : 8 * (int)sizeof(T);  // vector alignment needed
  const int vec_ok = job.channels == 1 && base_s % vb == 0 && base_d % vb == 0 &&
                     (job.src_pitch * sizeof(T)) % vb == 0 && (job.dst_pitch * sizeof(T)) % vb == 0;
  // grid.y is capped at 65535 row strips: tall narrow images get longer strips
  while ((job.out_h + L * R - 1) / (L * R) > 65535) R *= 2;
  dim3 grid((unsigned)(((n_tx + NT - 1) / NT) * job.channels),
            (unsigned)((job.out_h + L * R - 1) / (L * R)));
  med3_kernel<T><<<grid, NT, 0, stream>>>(job, (int)R, n_tx, vec_ok);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_med3(int bits, const Job& job, cudaStream_t s) {
  switch (bits) {
    case 8: return launch_med3_t<uint8_t>(job, s);
    case 16: return launch_med3_t<uint16_t>(job, s);
    default: return launch_med3_t<uint32_t>(job, s);
  }
}

}  // namespace tmb
