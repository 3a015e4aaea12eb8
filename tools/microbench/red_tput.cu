// Microbenchmark: shared-memory update throughput on sm_100a, the bound of
// the sliding-histogram kernels (tm_sweep.cuh).  Every lane updates its own
// column of a [bins][32] word array (the kernels' layout: a warp's accesses
// hit 32 distinct banks), with data-dependent bins.
//   RED     red.shared.add.u32 (no return)            -- the kernels' update
//   RED+1   red.shared.add.u32 with constant 1 (ptxas: ATOMS.POPC.INC)
//   LDS     ld.volatile.shared.u32 (the walk's loads)
//   RMW     ld + add + st (no atomics)
// Reports warp-instructions per clock per SM (timed with CUDA events over the
// whole grid, SM clock from nvidia-smi by the caller).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) bench(uint32_t* out, int iters) {
  __shared__ uint32_t hist[256 * 32];  // the warps of a CTA share one [256][32] array
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* h = hist;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(h + lane);
  // 16 data-dependent bins per lane, fixed across iterations: the timed loop
  // is nothing but the memory instructions
  uint32_t a[16];
  uint32_t x = lane * 2654435761u + blockIdx.x * 97u + warp;
#pragma unroll
  for (int u = 0; u < 16; u++) {
    x = x * 1664525u + 1013904223u;
    a[u] = base + ((x >> 24) * 32u) * 4u;
  }
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      if (MODE == 0) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[u]), "r"(x) : "memory");
      } else if (MODE == 1) {
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a[u]) : "memory");
      } else if (MODE == 2) {
        uint32_t v;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a[u]) : "memory");
        acc += v;
      } else {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a[u]) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a[u]), "r"(v + 1u) : "memory");
      }
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + hist[threadIdx.x];
}

template <int MODE>
void run(const char* name, int blocks_per_sm) {
  const int threads = 256, sms = 148, iters = 20000;
  const int blocks = sms * blocks_per_sm;
  uint32_t* out;
  cudaMalloc(&out, blocks * threads * 4);
  bench<MODE><<<blocks, threads>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<MODE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_ops = (double)blocks * (threads / 32) * iters * 16;
  const double per_s = warp_ops / (ms * 1e-3);
  printf("%-8s bps=%d  %8.3f ms  %7.2f T lane-ops/s  %6.3f warp-ops/clk/SM @1.965GHz  err=%s\n", name,
         blocks_per_sm, ms, per_s * 32 / 1e12, per_s / sms / 1.965e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int bps : {1, 2, 4}) {
    run<0>("RED", bps);
    run<1>("RED+1", bps);
    run<2>("LDS", bps);
    run<3>("RMW", bps);
  }
  return 0;
}
