// tm_rank_rect_u16_1.cu -- rectangular k_w x k_h instantiations of the rank
// kernel (tm_rank.cuh, run-time window height) for u16 and
// k_w in {5, 13, 21, 29, 37, 45, 53, 61, 69} (split so the build compiles in parallel).
#include "tm_rank.cuh"

namespace tmb {

int launch_rank_rect_u16_1(int kw, int kh, const Job& job, cudaStream_t s) {
  switch (kw) {
    case 5: return launch_rank_k<uint16_t, 5, true>(job, s, kh);
    case 13: return launch_rank_k<uint16_t, 13, true>(job, s, kh);
    case 21: return launch_rank_k<uint16_t, 21, true>(job, s, kh);
    case 29: return launch_rank_k<uint16_t, 29, true>(job, s, kh);
    case 37: return launch_rank_k<uint16_t, 37, true>(job, s, kh);
    case 45: return launch_rank_k<uint16_t, 45, true>(job, s, kh);
    case 53: return launch_rank_k<uint16_t, 53, true>(job, s, kh);
    case 61: return launch_rank_k<uint16_t, 61, true>(job, s, kh);
    case 69: return launch_rank_k<uint16_t, 69, true>(job, s, kh);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace tmb
