// tm_rank.cu -- entry points of the 16/32-bit data-aware kernel; the kernel
// lives in tm_rank.cuh, its instantiations in tm_rank_{u16,u32}_{0..3}.cu.
#include <cuda_runtime.h>

#include <mutex>

#include "tm_common.cuh"
#include "tm_kernels.h"

namespace tmb {

#ifdef TMB_RANK_PROFILE
void rank_prof_take_u16_0(unsigned long long* acc);
void rank_prof_take_u16_1(unsigned long long* acc);
void rank_prof_take_u16_2(unsigned long long* acc);
void rank_prof_take_u16_3(unsigned long long* acc);
void rank_prof_take_u32_0(unsigned long long* acc);
void rank_prof_take_u32_1(unsigned long long* acc);
void rank_prof_take_u32_2(unsigned long long* acc);
void rank_prof_take_u32_3(unsigned long long* acc);
extern "C" void tm_rank_profile(unsigned long long* out) {
  for (int i = 0; i < 8; i++) out[i] = 0;
  rank_prof_take_u16_0(out);
  rank_prof_take_u16_1(out);
  rank_prof_take_u16_2(out);
  rank_prof_take_u16_3(out);
  rank_prof_take_u32_0(out);
  rank_prof_take_u32_1(out);
  rank_prof_take_u32_2(out);
  rank_prof_take_u32_3(out);
}
#endif

int launch_rank_u16_0(int k, const Job& job, cudaStream_t s);
int launch_rank_u16_1(int k, const Job& job, cudaStream_t s);
int launch_rank_u16_2(int k, const Job& job, cudaStream_t s);
int launch_rank_u16_3(int k, const Job& job, cudaStream_t s);
int launch_rank_u32_0(int k, const Job& job, cudaStream_t s);
int launch_rank_u32_1(int k, const Job& job, cudaStream_t s);
int launch_rank_u32_2(int k, const Job& job, cudaStream_t s);
int launch_rank_u32_3(int k, const Job& job, cudaStream_t s);

int launch_rank_rect_u16_0(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u16_1(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u16_2(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u16_3(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u32_0(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u32_1(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u32_2(int kw, int kh, const Job& job, cudaStream_t s);
int launch_rank_rect_u32_3(int kw, int kh, const Job& job, cudaStream_t s);

// rectangular windows: width 3..75 (templated), height 3..127 (run time; the
// candidate positions keep footprint rows below 256: R + k_h - 1 <= 254)
bool rank_rect_supports(int bits, int kw, int kh) {
  return (bits == 16 || bits == 32) && kw >= 3 && kw <= 75 && (kw & 1) && kh >= 3 && kh <= 127 &&
         (kh & 1);
}

int launch_rank_rect(int bits, const Job& job, int kw, int kh, cudaStream_t s) {
  if (!rank_rect_supports(bits, kw, kh)) return (int)cudaErrorInvalidValue;
  const int part = ((kw - 3) / 2) % 4;
  if (bits == 16) {
    switch (part) {
      case 0: return launch_rank_rect_u16_0(kw, kh, job, s);
      case 1: return launch_rank_rect_u16_1(kw, kh, job, s);
      case 2: return launch_rank_rect_u16_2(kw, kh, job, s);
      default: return launch_rank_rect_u16_3(kw, kh, job, s);
    }
  }
  switch (part) {
    case 0: return launch_rank_rect_u32_0(kw, kh, job, s);
    case 1: return launch_rank_rect_u32_1(kw, kh, job, s);
    case 2: return launch_rank_rect_u32_2(kw, kh, job, s);
    default: return launch_rank_rect_u32_3(kw, kh, job, s);
  }
}

// The rank kernel's candidate staging comes from a private stream-ordered
// pool per device: freed blocks stay reserved between launches (up to 2 GB)
// without touching the device's default pool, which other users of
// cudaMallocAsync in the process (e.g. PyTorch) rely on.
namespace {
cudaMemPool_t stage_pool() {
  constexpr int kMaxDev = 64;
  constexpr uint64_t kKeepBytes = 2ull << 30;
  static std::mutex mu;
  static cudaMemPool_t pools[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
      cudaGetLastError();
      pools[dev] = nullptr;
      return nullptr;
    }
    uint64_t thr = kKeepBytes;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return pools[dev];
}
}  // namespace

void* rank_stage_alloc(size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = stage_pool();
  void* p = nullptr;
  if (!pool || cudaMallocFromPoolAsync(&p, bytes, pool, s) != cudaSuccess) {
    cudaGetLastError();  // no staging: the kernel places each group with its own scan
    return nullptr;
  }
  return p;
}

void rank_stage_free(void* p, cudaStream_t s) { cudaFreeAsync(p, s); }

bool rank_supports(int bits, int k) {
  // k <= 127: footprint rows (R + k - 1 <= 254) and columns (64 + k - 1)
  // stay below 256 in the candidates' 16-bit positions
  return (bits == 16 || bits == 32) && k >= 3 && k <= 127 && (k & 1);
}

int launch_rank(int bits, const Job& job, int k, cudaStream_t s) {
  if (!rank_supports(bits, k)) return (int)cudaErrorInvalidValue;
  const int part = ((k - 3) / 2) % 4;
  if (bits == 16) {
    switch (part) {
      case 0: return launch_rank_u16_0(k, job, s);
      case 1: return launch_rank_u16_1(k, job, s);
      case 2: return launch_rank_u16_2(k, job, s);
      default: return launch_rank_u16_3(k, job, s);
    }
  }
  switch (part) {
    case 0: return launch_rank_u32_0(k, job, s);
    case 1: return launch_rank_u32_1(k, job, s);
    case 2: return launch_rank_u32_2(k, job, s);
    default: return launch_rank_u32_3(k, job, s);
  }
}

}  // namespace tmb
