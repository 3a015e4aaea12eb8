// Microbenchmark: min/max instruction throughput on sm_100a (VIMNMX.U32,
// VIMNMX.U16x2, HMNMX2, mixes). Used to fix the ALU roofline denominator.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define MN(op, d, a, b) asm volatile(op " %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b))
template <int MODE>
__device__ __forceinline__ void ce(uint32_t& a, uint32_t& b) {
  uint32_t lo, hi;
  if (MODE == 0) { MN("min.u32", lo, a, b); MN("max.u32", hi, a, b); }
  else if (MODE == 1) { MN("min.u16x2", lo, a, b); MN("max.u16x2", hi, a, b); }
  else if (MODE == 2) { MN("min.f16x2", lo, a, b); MN("max.f16x2", hi, a, b); }
  a = lo; b = hi;
}
// MODE 3: half the CEs as u16x2, half as f16x2 (independent register sets)
template <int MODE, int N>
__global__ void __launch_bounds__(256) bench(uint32_t* out, int iters, long long* cyc) {
  uint32_t v[N];
#pragma unroll
  for (int i = 0; i < N; i++) v[i] = threadIdx.x * 7919u + i * 104729u + blockIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int s = 0; s < 4; s++) {
#pragma unroll
      for (int i = 0; i < N / 2; i++) {
        int a = (2 * i + (s & 1)) % N, b = (2 * i + 1 + (s & 1) + 2 * (s >> 1)) % N;
        if (a == b) continue;
        if (MODE == 3) { if (i & 1) ce<1>(v[a], v[b]); else ce<2>(v[a], v[b]); }
        else if (MODE == 4) { if (i & 1) ce<1>(v[a], v[b]); else ce<0>(v[a], v[b]); }
        else ce<MODE>(v[a], v[b]);
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < N; i++) acc ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int blocks_per_sm) {
  const int N = 16, threads = 256, sms = 148, iters = 200000;
  int blocks = sms * blocks_per_sm;
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  bench<MODE, N><<<blocks, threads>>>(out, 10, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<MODE, N><<<blocks, threads>>>(out, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long hc[4096]; cudaMemcpy(hc, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double avgc = 0; for (int i = 0; i < blocks; i++) avgc += hc[i]; avgc /= blocks;
  double instr = 2.0 * (N / 2) * 4 * iters * (double)blocks * threads;  // thread-level min/max instrs
  double per_s = instr / (ms * 1e-3);
  // cycles the SM spent: concurrent blocks share SM; per-SM instr/cycle:
  double per_sm_clk = instr / sms / (avgc);  // valid when all blocks co-resident
  printf("%-22s bps=%d  %.3f ms  %.2f T instr/s  %.1f instr/clk/SM (co-resident est)  clk~%.0f MHz  err=%s\n",
         name, blocks_per_sm, ms, per_s / 1e12, per_sm_clk, avgc / (ms * 1e-3) / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int bps : {4, 8}) {
    run<0>("u32 VIMNMX", bps);
    run<1>("u16x2 VIMNMX.U16x2", bps);
    run<2>("f16x2 HMNMX2", bps);
    run<3>("mix u16x2+f16x2", bps);
    run<4>("mix u16x2+u32", bps);
  }
  return 0;
}
