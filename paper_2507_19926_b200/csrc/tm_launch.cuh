// tm_launch.cuh -- host-side launch helpers shared by the generated launchers.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include "tm_oblivious.cuh"

namespace tmb {

// Raise the dynamic shared-memory limit of `fn` once per device.
template <typename F>
inline cudaError_t ensure_smem(F fn, int bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <typename T, int KW, int KH, int TW, int TH, int BX, int BY, class Prog, class CSort>
int launch_oblivious(const Job& job, cudaStream_t stream) {
  using Lay = OblLayout<T, KW, KH, TW, TH, BX, BY, Prog::kSpillSlots, Prog::kPair>;
  auto fn = obl_kernel<T, KW, KH, TW, TH, BX, BY, Prog, CSort>;
  cudaError_t e = ensure_smem(fn, Lay::kSmemBytes);
  if (e != cudaSuccess) return (int)e;
  static const int carve = [] {
    const char* v = getenv("TMB_CARVEOUT");
    return v ? atoi(v) : -1;
  }();
  if (carve >= 0) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  const int rows_per_cta = Lay::OH * Lay::kLanes;
  dim3 grid(((job.width + Lay::OW - 1) / Lay::OW) * job.channels,
            (job.out_h + rows_per_cta - 1) / rows_per_cta, 1);
  fn<<<grid, Lay::kThreads, Lay::kSmemBytes, stream>>>(job);
  return (int)cudaGetLastError();
}

}  // namespace tmb
