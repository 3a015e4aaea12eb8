// tm_kernels.h -- internal launcher declarations (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include "tm_common.cuh"

namespace tmb {

typedef int (*LaunchFn)(const Job&, cudaStream_t);

struct OblEntry {
  int bits;
  int k;
  int tw, th;
  LaunchFn fn;
};

int launch_select(int bits, const Job& job, int kw, int kh, cudaStream_t s);
int launch_aware(int bits, const Job& job, int k, cudaStream_t s);
bool hist8_supports(int k);
int launch_hist8(const Job& job, int k, cudaStream_t s);
bool hist8_rect_supports(int kw, int kh);
int launch_hist8_rect(const Job& job, int kw, int kh, cudaStream_t s);
bool rank_supports(int bits, int k);
int launch_rank(int bits, const Job& job, int k, cudaStream_t s);
bool rank_rect_supports(int bits, int kw, int kh);
// stream-ordered scratch for the rank kernel (private pool per device; NULL on failure)
void* rank_stage_alloc(size_t bytes, cudaStream_t s);
void rank_stage_free(void* p, cudaStream_t s);
int launch_rank_rect(int bits, const Job& job, int kw, int kh, cudaStream_t s);
int launch_med3(int bits, const Job& job, cudaStream_t s);

}  // namespace tmb
