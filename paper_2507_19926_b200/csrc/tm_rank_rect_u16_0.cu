// tm_rank_rect_u16_0.cu -- rectangular k_w x k_h instantiations of the rank
// kernel (tm_rank.cuh, run-time window height) for u16 and
// k_w in {3, 11, 19, 27, 35, 43, 51, 59, 67, 75} (split so the build compiles in parallel).
#include "tm_rank.cuh"

namespace tmb {

int launch_rank_rect_u16_0(int kw, int kh, const Job& job, cudaStream_t s) {
  switch (kw) {
    case 3: return launch_rank_k<uint16_t, 3, true>(job, s, kh);
    case 11: return launch_rank_k<uint16_t, 11, true>(job, s, kh);
    case 19: return launch_rank_k<uint16_t, 19, true>(job, s, kh);
    case 27: return launch_rank_k<uint16_t, 27, true>(job, s, kh);
    case 35: return launch_rank_k<uint16_t, 35, true>(job, s, kh);
    case 43: return launch_rank_k<uint16_t, 43, true>(job, s, kh);
    case 51: return launch_rank_k<uint16_t, 51, true>(job, s, kh);
    case 59: return launch_rank_k<uint16_t, 59, true>(job, s, kh);
    case 67: return launch_rank_k<uint16_t, 67, true>(job, s, kh);
    case 75: return launch_rank_k<uint16_t, 75, true>(job, s, kh);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace tmb
