// tm_rank_rect_u16_2.cu -- rectangular k_w x k_h instantiations of the rank
// kernel (tm_rank.cuh, run-time window height) for u16 and
// k_w in {7, 15, 23, 31, 39, 47, 55, 63, 71} (split so the build compiles in parallel).
#include "tm_rank.cuh"

namespace tmb {

int launch_rank_rect_u16_2(int kw, int kh, const Job& job, cudaStream_t s) {
  switch (kw) {
    case 7: return launch_rank_k<uint16_t, 7, true>(job, s, kh);
    case 15: return launch_rank_k<uint16_t, 15, true>(job, s, kh);
    case 23: return launch_rank_k<uint16_t, 23, true>(job, s, kh);
    case 31: return launch_rank_k<uint16_t, 31, true>(job, s, kh);
    case 39: return launch_rank_k<uint16_t, 39, true>(job, s, kh);
    case 47: return launch_rank_k<uint16_t, 47, true>(job, s, kh);
    case 55: return launch_rank_k<uint16_t, 55, true>(job, s, kh);
    case 63: return launch_rank_k<uint16_t, 63, true>(job, s, kh);
    case 71: return launch_rank_k<uint16_t, 71, true>(job, s, kh);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace tmb
