// tm_hist_rect.cu -- rectangular k_w x k_h instantiations of the 8-bit
// histogram kernel (tm_hist.cuh): the window width k_w is a template
// parameter (it sets the keys per lane and row), the height k_h a run-time
// value (ring rows, build rows, median rank).  Reference role: filter_image
// with a KernelSpec(k_w, k_h) (engine.py:24-25, geometry.py:25-58), which the
// reference routes to its oblivious engine; results are identical.
#include "tm_hist.cuh"

namespace tmb {
namespace {

template <int KW>
int launch_hist8_rect_k(const Job& job, int kh, cudaStream_t stream) {
  // 3 columns per lane while the counts fit 10-bit fields with a guard bit
  if constexpr (KW <= 21) {
    if (KW * kh < 512) return launch_hist8_t<KW, 3, true>(job, kh, stream);
  }
  return launch_hist8_t<KW, 2, true>(job, kh, stream);
}

template <int... Ks>
struct Hist8RectTable {
  static int launch(int kw, int kh, const Job& job, cudaStream_t s) {
    int rc = (int)cudaErrorInvalidValue;
    ((kw == Ks ? (rc = launch_hist8_rect_k<Ks>(job, kh, s), 0) : 0), ...);
    return rc;
  }
};

using Hist8RectAll = Hist8RectTable<3, 5, 7, 9, 11, 13, 15, 17, 19, 21, 23, 25, 27, 29, 31, 33, 35,
                                    37, 39, 41, 43, 45, 47, 49, 51, 53, 55, 57, 59, 61, 63, 65, 67,
                                    69, 71, 73, 75>;

}  // namespace

bool hist8_rect_supports(int kw, int kh) {
  return kw >= 3 && kw <= 75 && (kw & 1) && kh >= 3 && kh <= 127 && (kh & 1);
}

int launch_hist8_rect(const Job& job, int kw, int kh, cudaStream_t s) {
  if (!hist8_rect_supports(kw, kh)) return (int)cudaErrorInvalidValue;
  return Hist8RectAll::launch(kw, kh, job, s);
}

}  // namespace tmb
