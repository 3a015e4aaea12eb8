#include <cuda_fp16.h>
#include <cstdint>
__global__ void k_u32(const uint32_t* in, uint32_t* out){ uint32_t a=in[threadIdx.x], b=in[threadIdx.x+1], c=in[threadIdx.x+2];
  out[threadIdx.x]=min(a,b); out[threadIdx.x+64]=max(a,b); out[threadIdx.x+128]=__vimin3_u32(a,b,c); out[threadIdx.x+192]=__vimax3_u32(a,b,c);}
__global__ void k_u16x2(const uint32_t* in, uint32_t* out){ uint32_t a=in[threadIdx.x], b=in[threadIdx.x+1], c=in[threadIdx.x+2];
  out[threadIdx.x]=__vminu2(a,b); out[threadIdx.x+64]=__vmaxu2(a,b); out[threadIdx.x+128]=__vimin3_u16x2(a,b,c); out[threadIdx.x+192]=__vimax3_u16x2(a,b,c);}
__global__ void k_u8x4(const uint32_t* in, uint32_t* out){ uint32_t a=in[threadIdx.x], b=in[threadIdx.x+1];
  out[threadIdx.x]=__vminu4(a,b); out[threadIdx.x+64]=__vmaxu4(a,b);}
__global__ void k_h2(const __half2* in, __half2* out){ __half2 a=in[threadIdx.x], b=in[threadIdx.x+1];
  out[threadIdx.x]=__hmin2(a,b); out[threadIdx.x+64]=__hmax2(a,b);}
__global__ void k_f32(const float* in, float* out){ float a=in[threadIdx.x], b=in[threadIdx.x+1], c=in[threadIdx.x+2];
  out[threadIdx.x]=fminf(a,b); out[threadIdx.x+64]=fmaxf(fmaxf(a,b),c);}
