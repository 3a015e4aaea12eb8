// tm_rank_rect_u16_3.cu -- rectangular k_w x k_h instantiations of the rank
// kernel (tm_rank.cuh, run-time window height) for u16 and
// k_w in {9, 17, 25, 33, 41, 49, 57, 65, 73} (split so the build compiles in parallel).
#include "tm_rank.cuh"

namespace tmb {

int launch_rank_rect_u16_3(int kw, int kh, const Job& job, cudaStream_t s) {
  switch (kw) {
    case 9: return launch_rank_k<uint16_t, 9, true>(job, s, kh);
    case 17: return launch_rank_k<uint16_t, 17, true>(job, s, kh);
    case 25: return launch_rank_k<uint16_t, 25, true>(job, s, kh);
    case 33: return launch_rank_k<uint16_t, 33, true>(job, s, kh);
    case 41: return launch_rank_k<uint16_t, 41, true>(job, s, kh);
    case 49: return launch_rank_k<uint16_t, 49, true>(job, s, kh);
    case 57: return launch_rank_k<uint16_t, 57, true>(job, s, kh);
    case 65: return launch_rank_k<uint16_t, 65, true>(job, s, kh);
    case 73: return launch_rank_k<uint16_t, 73, true>(job, s, kh);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace tmb
