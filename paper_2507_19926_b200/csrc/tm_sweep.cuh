// tm_sweep.cuh -- the warp-level sliding-histogram sweep shared by the data-
// aware kernels (tm_hist.cuh: 8-bit samples, NB = 256 bins; tm_rank.cuh: 7-bit
// keys derived from 16/32-bit samples, NB = 128).
//
// One warp owns 32*CPL adjacent output columns; lane l owns columns CPL*l ..
// CPL*l + CPL-1, whose NB-bin histograms share storage: bin v of the lane's
// column c is bit field c (16 bits for CPL = 2, 10 bits for CPL = 3 when the
// window holds fewer than 512 samples) of one 32-bit word.  The window is K
// columns wide; its height only enters through the median rank (r2, set at
// init: (K * k_h + 1) / 2), so rectangular windows share the code.  A key at window column j (0..K+CPL-2
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
// Median tracking per column: m = bin holding rank r2, bl = #keys < m.  A row
// step applies the leaving and entering rows, updates bl with guard-bit-free
// SIMD byte compares (4 keys per IADD + LOP3 + dp4a) and walks m up to 8 bins
// per round trip for all CPL columns at once (packed-field arithmetic); the
// walk is warp-convergent (a converged lane's step is idempotent, so the lanes
// loop until all agree) and its per-column update is branch-free.
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

// CPL = output columns per lane sharing one count word: 2 (16-bit fields) or
// 3 (10-bit fields).  The walk needs the top bit of every field free, so
// counts must stay below 2^15 (K <= 181) or 2^9 (K <= 21).
template <int K, int NB = 256, int CPL = 2>
struct WarpSweep {
  static_assert(CPL == 2 || (CPL == 3 && K * K < 512), "counts must fit their fields");
  static constexpr int FB = CPL == 2 ? 16 : 10;     // bits per count field
  static constexpr uint32_t FM = (1u << FB) - 1u;
  static constexpr int kCPL = CPL;
  static constexpr int COLS = 32 * CPL;            // output columns per warp
  static constexpr int NS = K + CPL - 1;           // keys per lane per row
  static constexpr int NC = (NS + 3) / 4;          // 4-key chunks
  static constexpr int NWD = NC + 1;               // aligned words covering the chunks
#ifndef TMB_WALK_S
#define TMB_WALK_S 8  // bins per walk round trip (measured: 8)
#endif
  static constexpr int kWalk = TMB_WALK_S;
  static constexpr int kPad = kWalk > 8 ? kWalk : 8;  // zero bins below 0 / above NB - 1
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
  int r2;       // median rank (1-based): R2, or (K * kh + 1) / 2 for a K x kh window
  int m[CPL], bl[CPL];

  // `hist` = the warp's kHistBytes region.
  __device__ __forceinline__ void init(uint32_t* hist, int lane, int rank = R2) {
    hb = smem_u32(hist + kPad * 32 + lane);
    r2 = rank;
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
    // bl[c] += #entering < m[c] - #leaving < m[c] (before m moves).  Byte-wise
    // a < t without a guard bit: d = (a & 0x7F) + 0x80 - (t & 0x7F) per byte
    // (no borrow across bytes); a < t iff bit 7 of MAJ(~a, t, ~d).  The bytes
    // of the column's window are summed with dp4a (weights = the window mask),
    // 128 per key below the threshold.
    if constexpr (NB <= 128) {
      // 7-bit keys (the rank kernel): bit 7 of every byte is free, so
      // (a | 0x80) - t never borrows across bytes and its bit 7 is [a >= t];
      // the guard word is shared by every column
      uint32_t g_in[NC], g_out[NC];
#pragma unroll
      for (int i = 0; i < NC; i++) {
        g_in[i] = ci[i] | 0x80808080u;
        g_out[i] = co[i] | 0x80808080u;
      }
#pragma unroll
      for (int c = 0; c < CPL; c++) {
        const uint32_t tb = (uint32_t)m[c] * 0x01010101u;  // m <= 127 + kPad < 256
        int acc_i = 0, acc_o = 0;
#pragma unroll
        for (int i = 0; i < NC; i++) {
          const uint32_t mk = mask(c, i);
          if (mk) {
            const uint32_t li = ~(g_in[i] - tb) & 0x80808080u;
            const uint32_t lo = ~(g_out[i] - tb) & 0x80808080u;
            acc_i = (int)__dp4a(li, mk, (unsigned)acc_i);
            acc_o = (int)__dp4a(lo, mk, (unsigned)acc_o);
          }
        }
        bl[c] += (acc_i - acc_o) >> 7;
      }
    } else {
      uint32_t a_in[NC], a_out[NC];
#pragma unroll
      for (int i = 0; i < NC; i++) {
        a_in[i] = ci[i] & 0x7F7F7F7Fu;
        a_out[i] = co[i] & 0x7F7F7F7Fu;
      }
#pragma unroll
      for (int c = 0; c < CPL; c++) {
        const uint32_t tb = (uint32_t)m[c] * 0x01010101u;
        const uint32_t cb = 0x80808080u - (tb & 0x7F7F7F7Fu);
        int acc_i = 0, acc_o = 0;
#pragma unroll
        for (int i = 0; i < NC; i++) {
          const uint32_t mk = mask(c, i);
          if (mk) {
            const uint32_t di = a_in[i] + cb, dout = a_out[i] + cb;
            const uint32_t li = ((~ci[i] & tb) | (~ci[i] & ~di) | (tb & ~di)) & 0x80808080u;
            const uint32_t lo = ((~co[i] & tb) | (~co[i] & ~dout) | (tb & ~dout)) & 0x80808080u;
            acc_i = (int)__dp4a(li, mk, (unsigned)acc_i);
            acc_o = (int)__dp4a(lo, mk, (unsigned)acc_o);
          }
        }
        bl[c] += (acc_i - acc_o) >> 7;
      }
    }
    walk();
  }
  // Move m[c] to the bin holding rank R2, 8 bins per round trip, all columns
  // of the lane in one pass of packed-field (SWAR) arithmetic.  Column c scans
  // the window [s_c, s_c + 8): s_c = m_c going up (bl_c < R2), m_c - 8 going
  // down.  With B_c = #keys < s_c (bl_c, or bl_c minus the window total) and
  // P_j the packed prefix sums of the window's counts (P_0 = 0), the median
  // bin is s_c + n_c - 1 where n_c = #{j in 0..8 : P_j <= T_c},
  // T_c = R2 - 1 - B_c -- one comparison for all fields at once: with the
  // top bit of every field free (counts < 2^(FB-1)), (T | guards) - P keeps a
  // field's guard bit iff P <= T, and no borrow crosses fields.  n_c = 9 or
  // T_c < 0 mean the median lies beyond the window: the column moves 8 bins
  // on and the warp runs another round (a converged column's round is
  // idempotent, so the lanes loop until all agree).
  __device__ __forceinline__ void walk() {
    constexpr int S = kWalk;
    constexpr uint32_t ONE = CPL == 2 ? 0x00010001u : 0x00100401u;   // bit 0 of every field
    constexpr uint32_t GUARD = ONE << (FB - 1);
    for (;;) {
      int sc[CPL];
      uint32_t ac[CPL];
#pragma unroll
      for (int c = 0; c < CPL; c++) {
        sc[c] = bl[c] >= r2 ? m[c] - S : m[c];
        ac[c] = hb + (uint32_t)sc[c] * kBinStride;
      }
      uint32_t h[S], P[S + 1];
      P[0] = 0u;
#pragma unroll
      for (int j = 0; j < S; j++) {
        // field c from column c's load: a chain of bit selects (one LOP3 per
        // extra column; the bits above the top field are zero in every word)
        uint32_t x[CPL];
#pragma unroll
        for (int c = 0; c < CPL; c++) x[c] = ld_hist(ac[c] + j * kBinStride);
        uint32_t v = x[CPL - 1];
#pragma unroll
        for (int c = CPL - 2; c >= 0; c--) {
          constexpr uint32_t kAll = 0xFFFFFFFFu;
          const uint32_t lowc = kAll >> (32 - FB * (c + 1));  // fields 0..c
          v = (x[c] & lowc) | (v & ~lowc);
        }
        h[j] = v;
        P[j + 1] = P[j] + v;
      }
      int B[CPL], T[CPL];
      uint32_t Tp = GUARD;
#pragma unroll
      for (int c = 0; c < CPL; c++) {
        const int tot = (int)((P[S] >> (FB * c)) & FM);
        B[c] = bl[c] >= r2 ? bl[c] - tot : bl[c];
        T[c] = r2 - 1 - B[c];
        Tp |= (uint32_t)max(T[c], 0) << (FB * c);
      }
      uint32_t cnt = ONE, pin = 0u;  // j = 0: P_0 = 0 <= T
#pragma unroll
      for (int j = 1; j <= S; j++) {
        const uint32_t bits = ((Tp - P[j]) >> (FB - 1)) & ONE;
        cnt += bits;
        pin += h[j - 1] & (bits * FM);  // sum of h_i with P_{i+1} <= T: P_{n-1}
      }
      bool fin = true;
#pragma unroll
      for (int c = 0; c < CPL; c++) {  // branch-free: selects, no reconvergence
        const int n = (int)((cnt >> (FB * c)) & FM);
        const bool below = T[c] < 0;    // below the window: continue downwards from sc
        const bool above = n > S;       // above the window: continue upwards from sc + S
        const int add = above ? (int)((P[S] >> (FB * c)) & FM) : (int)((pin >> (FB * c)) & FM);
        m[c] = below ? sc[c] : sc[c] + (above ? S : n - 1);
        bl[c] = B[c] + (below ? 0 : add);
        fin = fin && !below && !above;
      }
      if (__all_sync(0xffffffffu, fin)) break;
    }
  }
};

}  // namespace tmb
