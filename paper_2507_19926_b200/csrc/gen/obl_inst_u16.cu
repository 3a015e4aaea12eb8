// generated -- oblivious kernel instantiations
#include "../tm_oblivious.cuh"
#include "../tm_launch.cuh"
#include "colsort.cuh"
#include "obl_k3_t2x2.cuh"
#include "obl_k5_t4x2.cuh"
#include "obl_k7_t4x2.cuh"
#include "obl_k9_t4x2.cuh"
#include "obl_k11_t4x2.cuh"
namespace tmb {
int launch_obl_u16_k3(const Job& job, cudaStream_t s) {
  return launch_oblivious<uint16_t, 3, 3, 2, 2, 64, 2, Prog_k3_t2x2, ColSort2>(job, s);
}
int launch_obl_u16_k5(const Job& job, cudaStream_t s) {
  return launch_oblivious<uint16_t, 5, 5, 4, 2, 32, 4, Prog_k5_t4x2, ColSort4>(job, s);
}
int launch_obl_u16_k7(const Job& job, cudaStream_t s) {
  return launch_oblivious<uint16_t, 7, 7, 4, 2, 32, 4, Prog_k7_t4x2, ColSort6>(job, s);
}
int launch_obl_u16_k9(const Job& job, cudaStream_t s) {
  return launch_oblivious<uint16_t, 9, 9, 4, 2, 32, 4, Prog_k9_t4x2, ColSort8>(job, s);
}
int launch_obl_u16_k11(const Job& job, cudaStream_t s) {
  return launch_oblivious<uint16_t, 11, 11, 4, 2, 32, 4, Prog_k11_t4x2, ColSort10>(job, s);
}
}  // namespace tmb
