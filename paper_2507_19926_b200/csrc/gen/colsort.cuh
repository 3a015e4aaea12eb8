// generated -- column sorting networks
#pragma once
#include <cstdint>
namespace tmb {
struct ColSort2 {
  template <class L>
  __device__ __forceinline__ static void run(uint32_t (&v)[2]) {
    { const uint32_t a = v[0], b = v[1]; v[0] = L::mn(a, b); v[1] = L::mx(a, b); }
  }
};
struct ColSort4 {
  template <class L>
  __device__ __forceinline__ static void run(uint32_t (&v)[4]) {
    { const uint32_t a = v[0], b = v[1]; v[0] = L::mn(a, b); v[1] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[3]; v[2] = L::mn(a, b); v[3] = L::mx(a, b); }
    { const uint32_t a = v[0], b = v[2]; v[0] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[3]; v[1] = L::mn(a, b); v[3] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[2]; v[1] = L::mn(a, b); v[2] = L::mx(a, b); }
  }
};
struct ColSort6 {
  template <class L>
  __device__ __forceinline__ static void run(uint32_t (&v)[6]) {
    { const uint32_t a = v[0], b = v[1]; v[0] = L::mn(a, b); v[1] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[3]; v[2] = L::mn(a, b); v[3] = L::mx(a, b); }
    { const uint32_t a = v[4], b = v[5]; v[4] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[0], b = v[2]; v[0] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[3]; v[1] = L::mn(a, b); v[3] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[2]; v[1] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[0], b = v[4]; v[0] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[5]; v[1] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[4]; v[2] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[5]; v[3] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[2]; v[1] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[4]; v[3] = L::mn(a, b); v[4] = L::mx(a, b); }
  }
};
struct ColSort8 {
  template <class L>
  __device__ __forceinline__ static void run(uint32_t (&v)[8]) {
    { const uint32_t a = v[0], b = v[1]; v[0] = L::mn(a, b); v[1] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[3]; v[2] = L::mn(a, b); v[3] = L::mx(a, b); }
    { const uint32_t a = v[4], b = v[5]; v[4] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[6], b = v[7]; v[6] = L::mn(a, b); v[7] = L::mx(a, b); }
    { const uint32_t a = v[0], b = v[2]; v[0] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[3]; v[1] = L::mn(a, b); v[3] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[2]; v[1] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[4], b = v[6]; v[4] = L::mn(a, b); v[6] = L::mx(a, b); }
    { const uint32_t a = v[5], b = v[7]; v[5] = L::mn(a, b); v[7] = L::mx(a, b); }
    { const uint32_t a = v[5], b = v[6]; v[5] = L::mn(a, b); v[6] = L::mx(a, b); }
    { const uint32_t a = v[0], b = v[4]; v[0] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[5]; v[1] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[6]; v[2] = L::mn(a, b); v[6] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[7]; v[3] = L::mn(a, b); v[7] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[4]; v[2] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[5]; v[3] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[2]; v[1] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[4]; v[3] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[5], b = v[6]; v[5] = L::mn(a, b); v[6] = L::mx(a, b); }
  }
};
struct ColSort10 {
  template <class L>
  __device__ __forceinline__ static void run(uint32_t (&v)[10]) {
    { const uint32_t a = v[0], b = v[1]; v[0] = L::mn(a, b); v[1] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[3]; v[2] = L::mn(a, b); v[3] = L::mx(a, b); }
    { const uint32_t a = v[4], b = v[5]; v[4] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[6], b = v[7]; v[6] = L::mn(a, b); v[7] = L::mx(a, b); }
    { const uint32_t a = v[8], b = v[9]; v[8] = L::mn(a, b); v[9] = L::mx(a, b); }
    { const uint32_t a = v[0], b = v[2]; v[0] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[3]; v[1] = L::mn(a, b); v[3] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[2]; v[1] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[4], b = v[6]; v[4] = L::mn(a, b); v[6] = L::mx(a, b); }
    { const uint32_t a = v[5], b = v[7]; v[5] = L::mn(a, b); v[7] = L::mx(a, b); }
    { const uint32_t a = v[5], b = v[6]; v[5] = L::mn(a, b); v[6] = L::mx(a, b); }
    { const uint32_t a = v[0], b = v[4]; v[0] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[5]; v[1] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[6]; v[2] = L::mn(a, b); v[6] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[7]; v[3] = L::mn(a, b); v[7] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[4]; v[2] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[5]; v[3] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[2]; v[1] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[4]; v[3] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[5], b = v[6]; v[5] = L::mn(a, b); v[6] = L::mx(a, b); }
    { const uint32_t a = v[0], b = v[8]; v[0] = L::mn(a, b); v[8] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[9]; v[1] = L::mn(a, b); v[9] = L::mx(a, b); }
    { const uint32_t a = v[4], b = v[8]; v[4] = L::mn(a, b); v[8] = L::mx(a, b); }
    { const uint32_t a = v[5], b = v[9]; v[5] = L::mn(a, b); v[9] = L::mx(a, b); }
    { const uint32_t a = v[2], b = v[4]; v[2] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[5]; v[3] = L::mn(a, b); v[5] = L::mx(a, b); }
    { const uint32_t a = v[6], b = v[8]; v[6] = L::mn(a, b); v[8] = L::mx(a, b); }
    { const uint32_t a = v[7], b = v[9]; v[7] = L::mn(a, b); v[9] = L::mx(a, b); }
    { const uint32_t a = v[1], b = v[2]; v[1] = L::mn(a, b); v[2] = L::mx(a, b); }
    { const uint32_t a = v[3], b = v[4]; v[3] = L::mn(a, b); v[4] = L::mx(a, b); }
    { const uint32_t a = v[5], b = v[6]; v[5] = L::mn(a, b); v[6] = L::mx(a, b); }
    { const uint32_t a = v[7], b = v[8]; v[7] = L::mn(a, b); v[8] = L::mx(a, b); }
  }
};
}  // namespace tmb
