// tm_hist.cu -- square k x k instantiations of the 8-bit histogram kernel
// (tm_hist.cuh).
#include "tm_hist.cuh"

namespace tmb {
namespace {

template <int K>
int launch_hist8_k(const Job& job, cudaStream_t stream) {
  // 3 columns per lane (10-bit fields) while K^2 < 512: a third fewer histogram
  // updates per output; the packed walk serves all columns at once
  return launch_hist8_t<K, (K <= 21 ? 3 : 2), false>(job, K, stream);
}

template <int... Ks>
struct Hist8Table {
  static int launch(int k, const Job& job, cudaStream_t s) {
    int rc = (int)cudaErrorInvalidValue;
    ((k == Ks ? (rc = launch_hist8_k<Ks>(job, s), 0) : 0), ...);
    return rc;
  }
};

#ifdef TMB_HIST_FEW_K  // experiment builds (tools/vbuild.py): a subset of k
using Hist8All = Hist8Table<15, 17, 21, 25, 33, 49, 75>;
#else
using Hist8All = Hist8Table<3, 5, 7, 9, 11, 13, 15, 17, 19, 21, 23, 25, 27, 29, 31, 33, 35, 37,
                            39, 41, 43, 45, 47, 49, 51, 53, 55, 57, 59, 61, 63, 65, 67, 69, 71,
                            73, 75, 77, 79, 81, 83, 85, 87, 89, 91, 93, 95, 97, 99, 101, 103,
                            105, 107, 109, 111, 113, 115, 117, 119, 121, 123, 125, 127>;
#endif

}  // namespace

bool hist8_supports(int k) { return k >= 3 && k <= 127 && (k & 1); }

int launch_hist8(const Job& job, int k, cudaStream_t s) {
  if (!hist8_supports(k)) return (int)cudaErrorInvalidValue;
  return Hist8All::launch(k, job, s);
}

}  // namespace tmb
