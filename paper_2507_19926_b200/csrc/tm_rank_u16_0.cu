// tm_rank_u16_0.cu -- instantiations of the rank kernel (tm_rank.cuh) for
// u16 and k in {3, 11, 19, 27, 35, 43, 51, 59, 67, 75, 83, 91, 99, 107, 115, 123}
// (split so the build compiles in parallel).
#include "tm_rank.cuh"

namespace tmb {

int launch_rank_u16_0(int k, const Job& job, cudaStream_t s) {
  switch (k) {
    case 3: return launch_rank_k<uint16_t, 3>(job, s);
    case 11: return launch_rank_k<uint16_t, 11>(job, s);
    case 19: return launch_rank_k<uint16_t, 19>(job, s);
    case 27: return launch_rank_k<uint16_t, 27>(job, s);
    case 35: return launch_rank_k<uint16_t, 35>(job, s);
    case 43: return launch_rank_k<uint16_t, 43>(job, s);
    case 51: return launch_rank_k<uint16_t, 51>(job, s);
    case 59: return launch_rank_k<uint16_t, 59>(job, s);
    case 67: return launch_rank_k<uint16_t, 67>(job, s);
    case 75: return launch_rank_k<uint16_t, 75>(job, s);
    case 83: return launch_rank_k<uint16_t, 83>(job, s);
    case 91: return launch_rank_k<uint16_t, 91>(job, s);
    case 99: return launch_rank_k<uint16_t, 99>(job, s);
    case 107: return launch_rank_k<uint16_t, 107>(job, s);
    case 115: return launch_rank_k<uint16_t, 115>(job, s);
    case 123: return launch_rank_k<uint16_t, 123>(job, s);
    default: return (int)cudaErrorInvalidValue;
  }
}

#ifdef TMB_RANK_PROFILE
void rank_prof_take_u16_0(unsigned long long* acc) {
  unsigned long long v[8], z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(v, g_rank_prof, sizeof(v));
  cudaMemcpyToSymbol(g_rank_prof, z, sizeof(z));
  for (int i = 0; i < 8; i++) acc[i] += v[i];
}
#endif

}  // namespace tmb
