// tm_rank_u16_2.cu -- instantiations of the rank kernel (tm_rank.cuh) for
// u16 and k in {7, 15, 23, 31, 39, 47, 55, 63, 71, 79, 87, 95, 103, 111, 119, 127}
// (split so the build compiles in parallel).
#include "tm_rank.cuh"

namespace tmb {

int launch_rank_u16_2(int k, const Job& job, cudaStream_t s) {
  switch (k) {
    case 7: return launch_rank_k<uint16_t, 7>(job, s);
    case 15: return launch_rank_k<uint16_t, 15>(job, s);
    case 23: return launch_rank_k<uint16_t, 23>(job, s);
    case 31: return launch_rank_k<uint16_t, 31>(job, s);
    case 39: return launch_rank_k<uint16_t, 39>(job, s);
    case 47: return launch_rank_k<uint16_t, 47>(job, s);
    case 55: return launch_rank_k<uint16_t, 55>(job, s);
    case 63: return launch_rank_k<uint16_t, 63>(job, s);
    case 71: return launch_rank_k<uint16_t, 71>(job, s);
    case 79: return launch_rank_k<uint16_t, 79>(job, s);
    case 87: return launch_rank_k<uint16_t, 87>(job, s);
    case 95: return launch_rank_k<uint16_t, 95>(job, s);
    case 103: return launch_rank_k<uint16_t, 103>(job, s);
    case 111: return launch_rank_k<uint16_t, 111>(job, s);
    case 119: return launch_rank_k<uint16_t, 119>(job, s);
    case 127: return launch_rank_k<uint16_t, 127>(job, s);
    default: return (int)cudaErrorInvalidValue;
  }
}

#ifdef TMB_RANK_PROFILE
void rank_prof_take_u16_2(unsigned long long* acc) {
  unsigned long long v[8], z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(v, g_rank_prof, sizeof(v));
  cudaMemcpyToSymbol(g_rank_prof, z, sizeof(z));
  for (int i = 0; i < 8; i++) acc[i] += v[i];
}
#endif

}  // namespace tmb
