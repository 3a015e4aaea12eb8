// tm_sweep.cuh -- the warp-level sliding-histogram sweep shared by the data-
// aware kernels (tm_hist.cu: 8-bit samples, NB = 256 bins; tm_rank.cu: 7-bit
// keys derived from 16/32-bit samples, NB = 128).
//
// One warp owns 32*CPL adjacent output columns; lane l owns columns CPL*l ..
// CPL*l + CPL-1, whose NB-bin histograms share storage: bin v of the lane's
// column c is bit field c (16 bits for CPL = 2, 10 bits for CPL = 3 when
// K^2 <= 1023) of one 32-bit word.  A key at window column j (0..K+CPL-2
// relative to the lane's first column) belongs to column c's window when
// c <= j < c + K, so its update is ONE shared-memory atomic add of a
// compile-time constant (e.g. 0x1 / 0x10001 / 0x10000 for CPL = 2) -- RED.ADD:
// no return, no read-modify-write round trip.  Counts are at most K^2 and
// never negative, so the fields never carry into each other.
//
// Histogram words: bins -kPad .. NB - 1 + kPad (zero padding for the 8-bin walk)
// x 32 lanes, word (bin, lane) at bin * 32 + lane -- a warp's accesses hit 32
// distinct banks whatever the bins.
//
// Median tracking per column: m = bin holding rank R2, bl = #keys < m.  A row
// step applies the leaving and entering rows, updates bl with SIMD byte
// compares (__vsetltu4: 4 keys per instruction) and walks m up to 8 bins per
// round trip; the walk is warp-convergent (a converged lane's step is
// idempotent, so the lanes loop until all agree).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Histogram traffic is explicit PTX (RED for updates, volatile loads/stores
// otherwise), so no compiler pass reorders accesses that alias through
// data-dependent bin addresses.
__device__ __forceinline__ void red_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_hist(uint32_t a) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_hist(uint32_t a, uint32_t v) {
  asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// CPL = output columns per lane sharing one count word: 2 (u16 fields, any K)
// or 3 (10-bit fields, K^2 <= 1023 i.e. K <= 31; measured slower).
template <int K, int NB = 256, int CPL = 2>
struct WarpSweep {
  static_assert(CPL == 2 || (CPL == 3 && K * K <= 1023), "counts must fit their fields");
  static constexpr int FB = CPL == 2 ? 16 : 10;     // bits per count field
  static constexpr uint32_t FM = (1u << FB) - 1u;
  static constexpr int kCPL = CPL;
  static constexpr int COLS = 32 * CPL;            // output columns per warp
  static constexpr int NS = K + CPL - 1;           // keys per lane per row
  static constexpr int NC = (NS + 3) / 4;          // 4-key chunks
  static constexpr int NWD = NC + 1;               // aligned words covering the chunks
  static constexpr int kPad = 8;                   // zero bins below 0 / above NB - 1
  static constexpr int kWords = NB + 2 * kPad;
  static constexpr int kHistBytes = kWords * 32 * 4;
  static constexpr int R2 = (K * K + 1) / 2;       // median rank, 1-based
  static constexpr uint32_t kBinStride = 4u * 32;

  // byte-lane flags of chunk i that belong to column c (samples c .. c+K-1)
  __host__ __device__ static constexpr uint32_t mask(int c, int i) {
    uint32_t m = 0;
    for (int b = 0; b < 4; b++)
      if (4 * i + b >= c && 4 * i + b < c + K) m |= 0x01u << (8 * b);
    return m;
  }
  // the update of a key at window column j: +1 in every column whose window holds it
  __host__ __device__ static constexpr uint32_t inc(int j) {
    uint32_t v = 0;
    for (int c = 0; c < CPL; c++)
      if (j >= c && j < c + K) v += 1u << (FB * c);
    return v;
  }

  uint32_t hb;  // shared address of bin 0 of this lane
  int m[CPL], bl[CPL];

  // `hist` = the warp's kHistBytes region.
  __device__ __forceinline__ void init(uint32_t* hist, int lane) {
    hb = smem_u32(hist + kPad * 32 + lane);
  }
  __device__ __forceinline__ void zero() {
    for (int b = -kPad; b < NB + kPad; b++) st_hist(hb + b * kBinStride, 0u);
  }
  // Keys 0..NS-1 of a byte row for this lane (row columns CPL*lane ..
  // CPL*lane + NS - 1), `row` 4-byte aligned, at least COLS + K + 8 bytes long.
  __device__ __forceinline__ static void chunks(const uint8_t* row, int lane, uint32_t (&ch)[NC]) {
    const int b0 = CPL * lane;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(row) + (b0 >> 2);
    const int sh = 8 * (b0 & 3);
    uint32_t w[NWD];
#pragma unroll
    for (int i = 0; i < NWD; i++) w[i] = wp[i];
#pragma unroll
    for (int i = 0; i < NC; i++) ch[i] = __funnelshift_r(w[i], w[i + 1], sh);
  }
  __device__ __forceinline__ uint32_t addr_of(const uint32_t (&ch)[NC], int j) const {
    return hb + __byte_perm(ch[j >> 2], 0u, 0x4440 | (j & 3)) * kBinStride;
  }
  __device__ __forceinline__ void add_row(const uint32_t (&ch)[NC]) {
#pragma unroll
    for (int j = 0; j < NS; j++) red_add(addr_of(ch, j), inc(j));
  }
  __device__ __forceinline__ int count(int b, int c) const {
    return (int)((ld_hist(hb + b * kBinStride) >> (FB * c)) & FM);
  }
  // After the K-row build: start every column at bin NB / 2.
  __device__ __forceinline__ void init_median() {
    int acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; c++) acc[c] = 0;
    for (int b = 0; b < NB / 2; b++) {
      const uint32_t w = ld_hist(hb + b * kBinStride);
#pragma unroll
      for (int c = 0; c < CPL; c++) acc[c] += (int)((w >> (FB * c)) & FM);
    }
#pragma unroll
    for (int c = 0; c < CPL; c++) {
      m[c] = NB / 2;
      bl[c] = acc[c];
    }
    walk();
  }
  // Slide the window one row: `co` leaves, `ci` enters.
  __device__ __forceinline__ void step(const uint32_t (&co)[NC], const uint32_t (&ci)[NC]) {
#pragma unroll
    for (int j = 0; j < NS; j++) {
      red_add(addr_of(co, j), 0u - inc(j));
      red_add(addr_of(ci, j), inc(j));
    }
    // bl[c] += #entering < m[c] - #leaving < m[c] (before m moves)
#pragma unroll
    for (int c = 0; c < CPL; c++) {
      const uint32_t mb = (uint32_t)m[c] * 0x01010101u;
      uint32_t ai = 0, ao = 0;
#pragma unroll
      for (int i = 0; i < NC; i++) {
        const uint32_t mk = mask(c, i);
        if (mk) {
          ai += __vsetltu4(ci[i], mb) & mk;
          ao += __vsetltu4(co[i], mb) & mk;
        }
      }
      bl[c] += (int)__dp4a(ai, 0x01010101u, 0u) - (int)__dp4a(ao, 0x01010101u, 0u);
    }
    walk();
  }
  // Move m[c] to the bin holding rank R2, 8 bins per round trip.
  //   up   (bl < R2):  prefix P_i = h(m) + .. + h(m+i); bins m .. m+i lie
  //                    wholly below rank R2 iff P_i <= X = R2 - 1 - bl;
  //                    with n = #{P_i <= X}: median bin m + n, bl += P_{n-1}.
  //   down (bl >= R2): P_i = h(m-1) + .. + h(m-1-i); bin m-1-i still holds
  //                    rank R2 or above iff P_i <= X = bl - R2; median bin
  //                    m - 1 - n, bl -= P_n.
  // n = 8 means keep going (m += / -= 8, bl +/-= P_7).
  __device__ __forceinline__ void walk() {
    constexpr int S = 8;
    for (;;) {
      bool fin[CPL];
#pragma unroll
      for (int c = 0; c < CPL; c++) {
        const bool down = bl[c] >= R2;
        const uint32_t a0 = hb + (uint32_t)(down ? m[c] - 1 : m[c]) * kBinStride;
        const uint32_t da = down ? (uint32_t)(-(int)kBinStride) : kBinStride;
        const int X = down ? bl[c] - R2 : R2 - 1 - bl[c];
        int P[S];
        int acc = 0;
#pragma unroll
        for (int i = 0; i < S; i++) {
          const uint32_t w = ld_hist(a0 + i * da);
          acc += (int)((w >> (FB * c)) & FM);
          P[i] = acc;
        }
        int n = 0, pin = 0, pout = P[S - 1];  // pin = P_{n-1} (0), pout = P_n (P_7)
#pragma unroll
        for (int i = S - 1; i >= 0; i--) {
          const bool le = P[i] <= X;
          n += le;
          pin = (le && pin == 0) ? P[i] : pin;    // largest P_i <= X (P monotone)
          pout = le ? pout : P[i];                // smallest P_i > X
        }
        fin[c] = n < S;
        if (down) {
          m[c] -= fin[c] ? n + 1 : S;
          bl[c] -= pout;
        } else {
          m[c] += n;
          bl[c] += pin;
        }
      }
      bool all = true;
#pragma unroll
      for (int c = 0; c < CPL; c++) all = all && fin[c];
      if (__all_sync(0xffffffffu, all)) break;
    }
  }
};

}  // namespace tmb
