// tm_select.cu -- brute-force window rank selection on the GPU.
//
// Serves variant="oracle" (the reference routes it to its brute-force filter,
// engine.py:40-41 / reference.py:26-43) and rectangular kernels: every output
// pixel independently selects the rank-(k_w*k_h+1)/2 value of its clamped
// window -- no tiling, no shared work -- by MSB-first radix selection: one
// counting pass over the window per bit of the data type.  O(k^2 * bits) per
// pixel; exact for any odd window up to 127 x 127 (shared-memory footprint).
#include "tm_common.cuh"
#include "tm_kernels.h"

namespace tmb {

constexpr int kSelTX = 32, kSelTY = 8;

template <typename T>
__global__ void __launch_bounds__(kSelTX * kSelTY)
select_kernel(Job job, int kw, int kh) {
  extern __shared__ uint32_t tile[];
  const int hw = kw / 2, hh = kh / 2;
  const int fw = kSelTX + kw - 1, fh = kSelTY + kh - 1;
  const int x0 = blockIdx.x * kSelTX, y0 = blockIdx.y * kSelTY;
  const int tid = threadIdx.y * kSelTX + threadIdx.x;
  for (int i = tid; i < fw * fh; i += kSelTX * kSelTY) {
    const int rx = i % fw, ry = i / fw;
    const int gx = clampi(x0 + rx - hw, 0, job.width - 1);
    const int gy = clampi(job.out_y0 + y0 + ry - hh, 0, job.src_h - 1);
    tile[i] = (uint32_t)load_px<T>(job, gy, gx);
  }
  __syncthreads();
  const int ox = x0 + threadIdx.x, oy = y0 + threadIdx.y;
  if (ox >= job.width || oy >= job.out_h) return;
  constexpr int kBits = 8 * sizeof(T);
  int rank = (kw * kh + 1) / 2;  // 1-based
  uint32_t prefix = 0;
  const uint32_t* win = tile + threadIdx.y * fw + threadIdx.x;
  for (int b = kBits - 1; b >= 0; b--) {
    int cnt = 0;  // window values agreeing with prefix on bits >= b (bit b = 0)
    for (int dy = 0; dy < kh; dy++) {
      const uint32_t* row = win + dy * fw;
      for (int dx = 0; dx < kw; dx++) cnt += ((row[dx] ^ prefix) >> b) == 0;
    }
    if (cnt < rank) {
      rank -= cnt;
      prefix |= 1u << b;
    }
  }
  store_px<T>(job, oy, ox, (T)prefix);
}

template <typename T>
static int launch_select_t(const Job& job, int kw, int kh, cudaStream_t s) {
  const int bytes = (kSelTX + kw - 1) * (kSelTY + kh - 1) * 4;
  auto fn = select_kernel<T>;
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return (int)e;
  }
  dim3 grid((job.width + kSelTX - 1) / kSelTX, (job.out_h + kSelTY - 1) / kSelTY, job.channels);
  fn<<<grid, dim3(kSelTX, kSelTY), bytes, s>>>(job, kw, kh);
  return (int)cudaGetLastError();
}

int launch_select(int bits, const Job& job, int kw, int kh, cudaStream_t s) {
  switch (bits) {
    case 8: return launch_select_t<uint8_t>(job, kw, kh, s);
    case 16: return launch_select_t<uint16_t>(job, kw, kh, s);
    default: return launch_select_t<uint32_t>(job, kw, kh, s);
  }
}

}  // namespace tmb
