// tm_rank_u32_3.cu -- instantiations of the rank kernel (tm_rank.cuh) for
// u32 and k in {9, 17, 25, 33, 41, 49, 57, 65, 73, 81, 89, 97, 105, 113, 121}
// (split so the build compiles in parallel).
#include "tm_rank.cuh"

namespace tmb {

int launch_rank_u32_3(int k, const Job& job, cudaStream_t s) {
  switch (k) {
    case 9: return launch_rank_k<uint32_t, 9>(job, s);
    case 17: return launch_rank_k<uint32_t, 17>(job, s);
    case 25: return launch_rank_k<uint32_t, 25>(job, s);
    case 33: return launch_rank_k<uint32_t, 33>(job, s);
    case 41: return launch_rank_k<uint32_t, 41>(job, s);
    case 49: return launch_rank_k<uint32_t, 49>(job, s);
    case 57: return launch_rank_k<uint32_t, 57>(job, s);
    case 65: return launch_rank_k<uint32_t, 65>(job, s);
    case 73: return launch_rank_k<uint32_t, 73>(job, s);
    case 81: return launch_rank_k<uint32_t, 81>(job, s);
    case 89: return launch_rank_k<uint32_t, 89>(job, s);
    case 97: return launch_rank_k<uint32_t, 97>(job, s);
    case 105: return launch_rank_k<uint32_t, 105>(job, s);
    case 113: return launch_rank_k<uint32_t, 113>(job, s);
    case 121: return launch_rank_k<uint32_t, 121>(job, s);
    default: return (int)cudaErrorInvalidValue;
  }
}

#ifdef TMB_RANK_PROFILE
void rank_prof_take_u32_3(unsigned long long* acc) {
  unsigned long long v[8], z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(v, g_rank_prof, sizeof(v));
  cudaMemcpyToSymbol(g_rank_prof, z, sizeof(z));
  for (int i = 0; i < 8; i++) acc[i] += v[i];
}
#endif

}  // namespace tmb
