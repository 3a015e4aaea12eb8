// tm_rank_u32_1.cu -- instantiations of the rank kernel (tm_rank.cuh) for
// u32 and k in {5, 13, 21, 29, 37, 45, 53, 61, 69, 77, 85, 93, 101, 109, 117, 125}
// (split so the build compiles in parallel).
#include "tm_rank.cuh"

namespace tmb {

int launch_rank_u32_1(int k, const Job& job, cudaStream_t s) {
  switch (k) {
    case 5: return launch_rank_k<uint32_t, 5>(job, s);
    case 13: return launch_rank_k<uint32_t, 13>(job, s);
    case 21: return launch_rank_k<uint32_t, 21>(job, s);
    case 29: return launch_rank_k<uint32_t, 29>(job, s);
    case 37: return launch_rank_k<uint32_t, 37>(job, s);
    case 45: return launch_rank_k<uint32_t, 45>(job, s);
    case 53: return launch_rank_k<uint32_t, 53>(job, s);
    case 61: return launch_rank_k<uint32_t, 61>(job, s);
    case 69: return launch_rank_k<uint32_t, 69>(job, s);
    case 77: return launch_rank_k<uint32_t, 77>(job, s);
    case 85: return launch_rank_k<uint32_t, 85>(job, s);
    case 93: return launch_rank_k<uint32_t, 93>(job, s);
    case 101: return launch_rank_k<uint32_t, 101>(job, s);
    case 109: return launch_rank_k<uint32_t, 109>(job, s);
    case 117: return launch_rank_k<uint32_t, 117>(job, s);
    case 125: return launch_rank_k<uint32_t, 125>(job, s);
    default: return (int)cudaErrorInvalidValue;
  }
}

#ifdef TMB_RANK_PROFILE
void rank_prof_take_u32_1(unsigned long long* acc) {
  unsigned long long v[8], z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(v, g_rank_prof, sizeof(v));
  cudaMemcpyToSymbol(g_rank_prof, z, sizeof(z));
  for (int i = 0; i < 8; i++) acc[i] += v[i];
}
#endif

}  // namespace tmb
