// tm_rank.cu -- entry points of the 16/32-bit data-aware kernel; the kernel
// lives in tm_rank.cuh, its instantiations in tm_rank_{u16,u32}_{0..3}.cu.
#include <cuda_runtime.h>

#include "tm_common.cuh"
#include "tm_kernels.h"

namespace tmb {

#ifdef TMB_RANK_PROFILE
void rank_prof_take_u16_0(unsigned long long* acc);
void rank_prof_take_u16_1(unsigned long long* acc);
void rank_prof_take_u16_2(unsigned long long* acc);
void rank_prof_take_u16_3(unsigned long long* acc);
void rank_prof_take_u32_0(unsigned long long* acc);
void rank_prof_take_u32_1(unsigned long long* acc);
void rank_prof_take_u32_2(unsigned long long* acc);
void rank_prof_take_u32_3(unsigned long long* acc);
extern "C" void tm_rank_profile(unsigned long long* out) {
  for (int i = 0; i < 8; i++) out[i] = 0;
  rank_prof_take_u16_0(out);
  rank_prof_take_u16_1(out);
  rank_prof_take_u16_2(out);
  rank_prof_take_u16_3(out);
  rank_prof_take_u32_0(out);
  rank_prof_take_u32_1(out);
  rank_prof_take_u32_2(out);
  rank_prof_take_u32_3(out);
}
#endif

int launch_rank_u16_0(int k, const Job& job, cudaStream_t s);
int launch_rank_u16_1(int k, const Job& job, cudaStream_t s);
int launch_rank_u16_2(int k, const Job& job, cudaStream_t s);
int launch_rank_u16_3(int k, const Job& job, cudaStream_t s);
int launch_rank_u32_0(int k, const Job& job, cudaStream_t s);
int launch_rank_u32_1(int k, const Job& job, cudaStream_t s);
int launch_rank_u32_2(int k, const Job& job, cudaStream_t s);
int launch_rank_u32_3(int k, const Job& job, cudaStream_t s);

bool rank_supports(int bits, int k) {
  return (bits == 16 || bits == 32) && k >= 3 && k <= 75 && (k & 1);
}

int launch_rank(int bits, const Job& job, int k, cudaStream_t s) {
  if (!rank_supports(bits, k)) return (int)cudaErrorInvalidValue;
  const int part = ((k - 3) / 2) % 4;
  if (bits == 16) {
    switch (part) {
      case 0: return launch_rank_u16_0(k, job, s);
      case 1: return launch_rank_u16_1(k, job, s);
      case 2: return launch_rank_u16_2(k, job, s);
      default: return launch_rank_u16_3(k, job, s);
    }
  }
  switch (part) {
    case 0: return launch_rank_u32_0(k, job, s);
    case 1: return launch_rank_u32_1(k, job, s);
    case 2: return launch_rank_u32_2(k, job, s);
    default: return launch_rank_u32_3(k, job, s);
  }
}

}  // namespace tmb
