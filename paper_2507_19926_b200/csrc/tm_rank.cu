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

int launch_rank_rect_u16_0(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u16_1(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u16_2(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u16_3(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u32_0(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u32_1(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u32_2(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u32_3(int kw, int kh, const Job& job, cudaStream_t s);

// rectangular windows: width 3..75 (templated), height 3..127 (run time; the
// candidate positions keep footprint rows below 256: R + k_h - 1 <= 254)
bool rank_rect_supports(int bits, int kw, int kh) {
  return (bits == 16 || bits == 32) && kw >= 3 && kw <= 75 && (kw & 1) && kh >= 3 && kh <= 127 &&
         (kh & 1);
}

int launch_rank_rect(int bits, const Job& job, int kw, int kh, cudaStream_t s) {
  if (!rank_rect_supports(bits, kw, kh)) return (int)cudaErrorInvalidValue;
  const int part = ((kw - 3) / 2) % 4;
  if (bits == 16) {
    switch (part) {
      case 0: return launch_rank_rect_u16_0(kw, kh, job, s);
      case 1: return launch_rank_rect_u16_1(kw, kh, job, s);
      case 2: return launch_rank_rect_u16_2(kw, kh, job, s);
      default: return launch_rank_rect_u16_3(kw, kh, job, s);
    }
  }
  switch (part) {
    case 0: return launch_rank_rect_u32_0(kw, kh, job, s);
    case 1: return launch_rank_rect_u32_1(kw, kh, job, s);
    case 2: return launch_rank_rect_u32_2(kw, kh, job, s);
    default: return launch_rank_rect_u32_3(kw, kh, job, s);
  }
}

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
