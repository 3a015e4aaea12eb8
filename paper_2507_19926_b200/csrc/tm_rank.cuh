// tm_rank.cuh -- data-aware O(k) median for 16- and 32-bit images (variant (2)
// for uint16 / uint32): the sliding-histogram sweep (tm_sweep.cuh) run twice
// on 7-bit KEYS derived from the samples.
//
// Reference role: the data-aware engine (aware.py:437-492) -- the candidates
// for a tile of outputs are narrowed with a cheap pass, then the median is
// selected exactly by rank among the survivors (the paper's forgetful
// candidate windows, section 5.1, applied per tile of outputs).
//
// One warp = one work item: 64 output columns x up to RMAX output rows.  Every
// pass is a sweep of the shared sliding histogram (tm_sweep.cuh) over 7-bit
// keys; what changes between passes is the key function (KeyFn below):
//  * range sweep: key = the position of each sample inside the footprint's own
//    value range [fmin, fmax] (7 bits) -> every median of the item lies in the
//    union [lo, hi] of the bins the pixels' walks end in;
//  * candidate fine sweep (few samples inside an interval [lo, hi]): keys 0
//    below lo, 127 above hi, 1 + floor((v - lo) * 126 / span) inside; the
//    candidates are bucketed by key and sorted, so the walk's bucket plus its
//    residual rank picks the median among the bucket's in-window candidates;
//  * exact slices (one value per bin over 126 values): the walk's bin is the
//    median.
// Exact by construction for every input; the per-item decisions are described
// above rank_kernel.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <type_traits>

#include "tm_common.cuh"
#include "tm_kernels.h"
#include "tm_sweep.cuh"

namespace tmb {
namespace {

template <typename T, int K>
struct RankCfg {
  static constexpr int NB = 128;                       // key bins (7-bit keys)
  using SW = WarpSweep<K, NB>;
#ifndef TMB_RANK_BIG_RMAX
#define TMB_RANK_BIG_RMAX 128
#endif
  static constexpr int RMAX = K <= 45 ? 128 : TMB_RANK_BIG_RMAX;
#ifndef TMB_RANK_G
#define TMB_RANK_G 1  // measured: G = 4 -> 1 is +8..58 % (fewer prefetch registers)
#endif
  static constexpr int G = TMB_RANK_G;                 // ring refill group (rows)
  static constexpr int H = K / 2;
  static constexpr int FW = 64 + K - 1;                // footprint columns
  static constexpr int KW = ((FW + 3) / 4) * 4 + 8;    // ring row bytes
  static constexpr int RING = K + 2 * G + 1;           // ring rows
  static constexpr int kRingBytes = ((RING * KW + 15) / 16) * 16;
  // candidates per (sub-)item: the median spread of a 64 x 128 item (and so
  // the candidate count) grows with k; small k buys occupancy with less
#ifndef TMB_RANK_BIG_CMAX
#define TMB_RANK_BIG_CMAX 4096
#endif
  static constexpr int CMAX =
      K <= 45 ? 2048 : (sizeof(T) == 2 && K <= 53 ? 3072 : TMB_RANK_BIG_CMAX);  // measured
  static constexpr int kValBytes = CMAX * (int)sizeof(T);
  static constexpr int kPosBytes = CMAX * 2;
  static constexpr int kStack = 16;                    // pending value intervals
  static constexpr int kStartBytes = ((NB + 1) + 3 * kStack + 3) * 4;  // start[], interval stack
  static constexpr int kHistBytes = SW::kHistBytes;
  static constexpr int kWarpBytes = kHistBytes + kRingBytes + kValBytes + kPosBytes + kStartBytes;
  static constexpr int E = (G * FW + 31) / 32;         // prefetch samples per lane
};

template <typename T>
__device__ __forceinline__ uint32_t load_s(const T* src, const Job& job, int y, int x) {
  return __ldg(src + (int64_t)y * job.src_pitch + (int64_t)x * job.channels);
}

// Key of a sample.
//   f < 0  (range pass):    (v - lo) >> shift clamped to [0, NB-1] -- the 7-bit
//                           position of v inside a guess of the footprint's own
//                           value range (adaptive: narrow or smooth data
//                           spreads over all bins; outliers clamp to the ends);
//   f == 0 (exact slice):   0 below lo, NB-1 above hi, 1 + v - lo inside (one
//                           value per bin, hi - lo <= NB - 3);
//   f > 0  (interval pass): 0 / NB-1 outside [lo, hi], 1 + floor((v - lo) *
//                           (NB - 2) / span) inside (monotone in v).
// The mode F is a template parameter: every sweep / scan is compiled for the
// key function it uses (no per-sample mode branches).
template <int NB, int F>
struct KeyFn {
  uint32_t lo, hi;
  uint32_t mul;  // f > 0: bin = (v - lo) * mul >> 32, all NB - 2 inner bins in use
  int shift;
  __device__ __forceinline__ uint8_t operator()(uint32_t v) const {
    if constexpr (F < 0) {
      return v < lo ? 0 : (uint8_t)min((v - lo) >> shift, (uint32_t)(NB - 1));
    } else {
      if (v < lo) return 0;
      if (v > hi) return NB - 1;
      return (uint8_t)(1 + (F == 0 ? v - lo : __umulhi(v - lo, mul)));
    }
  }  // f > 0: the smallest value whose key is >= b (1 <= b <= NB - 1); hi + 1
  // (mod 2^32) when no value of [lo, hi] gets there.  Exact: key(v) >= b iff
  // (v - lo) * mul >= (b - 1) * 2^32.
  __device__ __forceinline__ uint32_t first_of(int b) const {
    const uint64_t d = (((uint64_t)(b - 1) << 32) + mul - 1) / mul;
    return d <= (uint64_t)(hi - lo) ? lo + (uint32_t)d : hi + 1u;
  }
};

__device__ __forceinline__ uint32_t warp_min(uint32_t v) {
  return __reduce_min_sync(0xffffffffu, v);
}
__device__ __forceinline__ uint32_t warp_max(uint32_t v) {
  return __reduce_max_sync(0xffffffffu, v);
}

#ifdef TMB_RANK_PROFILE
static __device__ unsigned long long g_rank_prof[8];  // per translation unit; tm_rank.cu sums them
#define RANK_T(i) do { const long long _n = clock64(); if (lane == 0) atomicAdd(&g_rank_prof[i], (unsigned long long)(_n - _t)); _t = _n; } while (0)
#else
#define RANK_T(i) do { } while (0)
#endif

// Per item (64 columns x R output rows) the kernel finds value intervals that
// hold every median of the item and resolves each exactly, the cheapest way
// the scans' counts allow -- so smooth, constant, narrow-range and impulse
// data cost a small constant factor of random data, never a per-pixel path:
//   0. footprint scan: [fmin, fmax].  At most NB - 2 distinct values -> one
//      exact slice sweep (constant and near-constant data);
//   1. range sweep on 7-bit positions in [fmin, fmax] -> the interval [lo, hi]
//      of the bins the medians landed in;
//   2. per interval: count scan of its candidates (samples inside) over 126
//      fine buckets.  If they fit (CMAX): place, sort, fine sweep (random-like
//      data: concentrated medians).  Otherwise the medians are spread: exact
//      slices of 126 values when the candidates' range is short (gradients,
//      impulse noise over them); a recount when that range is much narrower;
//      else consecutive buckets are grouped to fit CMAX, one fine sweep per
//      group, and a bucket that alone overflows becomes an interval of its own
//      (126 finer buckets; intervals pend on a small stack).
// Every pixel's median lies in exactly one resolved bucket or slice, and each
// pass stores only the pixels whose median it resolves.
// K = window width; the height is K (square) or the run-time kh_rt (RT,
// rectangular K x kh windows, tm_rank_rect_*.cu): it sets the ring rows, the
// build rows, the row test of a candidate and the median rank.
template <typename T, int K, bool RT>
__global__ void __launch_bounds__(32, 1)
    rank_kernel(Job job, int R, int n_strips, int n_segs, int kh_rt, uint8_t* gstage,
                int64_t gstride, int gcap) {
  using C = RankCfg<T, K>;
  using SW = typename C::SW;
  constexpr int NB = C::NB;
  constexpr uint32_t kInner = NB - 2;  // inner bins of a key
  constexpr int kStack = C::kStack;
  extern __shared__ __align__(16) uint32_t smem[];
  const int KH = RT ? kh_rt : K;                    // window height
  const int RING = RT ? KH + 2 * C::G + 1 : C::RING;
  const int ring_bytes = RT ? ((RING * C::KW + 15) / 16) * 16 : C::kRingBytes;
  const int lane = threadIdx.x;
  uint8_t* ring = reinterpret_cast<uint8_t*>(smem) + C::kHistBytes;
  T* cval = reinterpret_cast<T*>(ring + ring_bytes);                     // bucketed candidates
  uint16_t* cpos = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(cval) + C::kValBytes);
  int* start = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(cpos) + C::kPosBytes);
  uint32_t* stk = reinterpret_cast<uint32_t*>(start + NB + 1);          // interval stack
  int* cur = reinterpret_cast<int*>(smem);  // placement cursors: idle histogram words
  // this warp's global staging of spread candidates (gcap entries), or none
  T* gval = gstage ? reinterpret_cast<T*>(gstage + (int64_t)blockIdx.x * gstride) : nullptr;
  uint16_t* gpos = gstage ? reinterpret_cast<uint16_t*>(gval + gcap) : nullptr;
  SW sw;
  sw.init(smem, lane, (K * KH + 1) / 2);
  const int W = job.width, SH = job.src_h, CH = job.channels;
  const int n_items = n_strips * CH * n_segs;

  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int chan = item % CH;
    const int strip = (item / CH) % n_strips;
    const int seg = item / (CH * n_strips);
    const int X0 = strip * 64;
    const int Yi = seg * R;
    const int rows_item = min(R, job.out_h - Yi);
    const T* src = static_cast<const T*>(job.src) + chan;
    T* dst = static_cast<T*>(job.dst) + chan;
    const int x = X0 + 2 * lane;

    {
      const int rows = rows_item;
      const int Y0 = Yi;
      const int sy_base = job.out_y0 + Y0 - KH / 2;  // source row of footprint row 0
      const int q_end = KH + rows - 1;               // footprint rows
#ifdef TMB_RANK_PROFILE
      long long _t = clock64();
#endif

      // G footprint rows of samples [q0, q0 + G) into registers.  Slot e of
      // a lane reads group row g_e at footprint column c_e; both and the
      // clamped column offset are fixed per item (computed once here).
      int g_of[C::E], xo[C::E], c_of[C::E];
#pragma unroll
      for (int e = 0; e < C::E; e++) {
        const int idx = lane + e * 32;
        const int g = idx / C::FW, c = idx - g * C::FW;
        g_of[e] = idx < C::G * C::FW ? g : 0x3fffffff;  // an unused slot never passes q < q_end
        xo[e] = clampi(X0 - C::H + c, 0, W - 1) * CH;
        c_of[e] = c;
      }
      auto fetch_raw = [&](int q0, uint32_t (&v)[C::E]) {
        if constexpr (C::G == 1) {  // one footprint row: one row pointer per fetch
          const T* rp = src + (int64_t)clampi(sy_base + q0, 0, SH - 1) * job.src_pitch;
          const bool row_ok = q0 < q_end;
#pragma unroll
          for (int e = 0; e < C::E; e++) v[e] = (row_ok && g_of[e] == 0) ? __ldg(rp + xo[e]) : 0u;
        } else {
#pragma unroll
          for (int e = 0; e < C::E; e++) {
            v[e] = 0u;
            if (q0 + g_of[e] < q_end) {
              const int sy = clampi(sy_base + q0 + g_of[e], 0, SH - 1);
              v[e] = __ldg(src + (int64_t)sy * job.src_pitch + xo[e]);
            }
          }
        }
      };
      auto valid = [&](int q0, int e) { return q0 + g_of[e] < q_end; };
      auto pos_of = [&](int q0, int e) { return (uint32_t)(((q0 + g_of[e]) << 8) | c_of[e]); };

      // One sweep over the sub-item with keys from `kf`; `emit(t)` after each row.
      uint32_t fmin = 0xFFFFFFFFu, fmax = 0u;  // the footprint's value range (lane-partial)
      auto sweep = [&](const auto& kf, auto&& emit, bool track = false) {
        auto stash = [&](int q0, const uint32_t (&v)[C::E]) {
          uint8_t* rb = ring + (q0 % RING) * C::KW;  // G = 1: one ring row
#pragma unroll
          for (int e = 0; e < C::E; e++) {
            if (valid(q0, e)) {
              uint8_t* dstp = C::G == 1 ? rb + c_of[e]
                                        : ring + ((q0 + g_of[e]) % RING) * C::KW + c_of[e];
              *dstp = kf(v[e]);
              if (track) {  // every footprint sample is stashed exactly once
                fmin = min(fmin, v[e]);
                fmax = max(fmax, v[e]);
              }
            }
          }
        };
        auto row = [&](int q) { return ring + (q % RING) * C::KW; };
        __syncwarp();
        {
          // prologue: rows [0, K + G), loads double-buffered against stores
          uint32_t va[C::E], vb[C::E];
          fetch_raw(0, va);
          int q = 0;
          for (; q + C::G < KH + C::G; q += 2 * C::G) {
            fetch_raw(q + C::G, vb);
            stash(q, va);
            if (q + 2 * C::G < KH + C::G) fetch_raw(q + 2 * C::G, va);
            stash(q + C::G, vb);
          }
          if (q < KH + C::G) stash(q, va);
        }
        sw.zero();
        __syncwarp();
        for (int q = 0; q < KH; q++) {
          uint32_t ch[SW::NC];
          SW::chunks(row(q), lane, ch);
          sw.add_row(ch);
        }
        sw.init_median();
        emit(0);
        // ring rows of the leaving / entering footprint rows, advanced with a
        // wrap instead of a modulo per step
        const uint8_t* ring_end = ring + RING * C::KW;
        const uint8_t* po = row(0);
        const uint8_t* pi = row(KH);
        for (int t0 = 1; t0 < rows; t0 += C::G) {
          uint32_t nxt[C::E];
          const int qn = KH + t0 - 1 + C::G;
          if (qn < q_end) fetch_raw(qn, nxt);
          const int t1 = min(t0 + C::G, rows);
          for (int t = t0; t < t1; t++) {
            uint32_t co[SW::NC], ci[SW::NC];
            SW::chunks(po, lane, co);
            SW::chunks(pi, lane, ci);
            po += C::KW;
            pi += C::KW;
            if (po == ring_end) po = ring;
            if (pi == ring_end) pi = ring;
            sw.step(co, ci);
            emit(t);
          }
          if (qn < q_end) stash(qn, nxt);
          __syncwarp();
        }
      };
      // Every EVERY-th footprint row (G = 1): visit(v, pos).
      auto scan_rows = [&](int every, auto&& visit) {
        for (int q0 = 0; q0 < q_end; q0 += every) {
          uint32_t va[C::E];
          fetch_raw(q0, va);
#pragma unroll
          for (int e = 0; e < C::E; e++)
            if (valid(q0, e)) visit(va[e], pos_of(q0, e));
        }
      };
      // Every footprint sample once (loads double-buffered): visit(v, pos).
      auto scan = [&](auto&& visit) {
        uint32_t va[C::E], vb[C::E];
        fetch_raw(0, va);
        auto visit_all = [&](int q0, const uint32_t (&v)[C::E]) {
#pragma unroll
          for (int e = 0; e < C::E; e++)
            if (valid(q0, e)) visit(v[e], pos_of(q0, e));
        };
        int q0 = 0;
        for (; q0 + C::G < q_end; q0 += 2 * C::G) {
          fetch_raw(q0 + C::G, vb);
          visit_all(q0, va);
          if (q0 + 2 * C::G < q_end) fetch_raw(q0 + 2 * C::G, va);
          visit_all(q0 + C::G, vb);
        }
        if (q0 < q_end) visit_all(q0, va);
      };
      auto put = [&](int t, int c, uint32_t v) {
        if (x + c < W) dst[(int64_t)(Y0 + t) * job.dst_pitch + (int64_t)(x + c) * CH] = (T)v;
      };
      // Bins [blo, bhi] holding the medians of the sub-item's in-image columns.
      // Only inner bins count: a pixel whose walk ends in bin 0 / NB-1 has its
      // median outside the swept interval, so another interval resolves it
      // (counting those bins would grow the next interval back to the
      // footprint's range, and the work-list could cycle).  blo > bhi: no
      // median inside.
      auto range_pass = [&](const auto& kf, int& blo, int& bhi) {
        int b0 = NB - 1, b1 = 0;
        sweep(kf, [&](int) {
#pragma unroll
          for (int c = 0; c < 2; c++) {
            const int b = sw.m[c];
            if (x + c < W && b >= 1 && b <= NB - 2) {
              b0 = min(b0, b);
              b1 = max(b1, b);
            }
          }
        });
        blo = (int)warp_min((uint32_t)b0);
        bhi = (int)warp_max((uint32_t)b1);
      };
      // Exact slice: one value per bin over [a, b] (b - a < NB - 2); stores
      // every pixel whose median lies in [a, b].
      auto slice = [&](uint32_t a, uint32_t b) {
        const KeyFn<NB, 0> kx{a, b, 0u, 0};
        sweep(kx, [&](int t) {
#pragma unroll
          for (int c = 0; c < 2; c++) {
            const int bb = sw.m[c];
            if (bb >= 1 && bb <= NB - 2) put(t, c, a + (uint32_t)(bb - 1));
          }
        });
      };
      auto slices = [&](uint32_t a, uint32_t b) {
        for (uint64_t s0 = a; s0 <= b; s0 += kInner)
          slice((uint32_t)s0, (uint32_t)min((uint64_t)b, s0 + kInner - 1));
      };

      // Candidates of buckets [ba, bb] of `kf` (they fit: start[bb + 1] -
      // start[ba] <= CMAX): place them, sort each bucket by value, run the fine
      // sweep; stores every pixel whose median lies in those buckets -- its
      // walk ends in bucket b with residual rank R2 - #keys < b, and the median
      // is that rank among b's in-window candidates in sorted order.
      // Candidates of buckets [ba, bb] of `kf` into cval / cpos: `from_global`
      // copies them from the item's global staging (placed there by one scan
      // for every bucket, below), else one placement scan of the footprint.
      auto resolve = [&](const auto& kf, int ba, int bb, bool from_global = false) {
        const int base = start[ba];
        if (from_global) {
          const int n = start[bb + 1] - base;
          for (int i = lane; i < n; i += 32) {  // contiguous, coalesced
            cval[i] = gval[base + i];
            cpos[i] = gpos[base + i];
          }
        } else {
          for (int b = ba + lane; b <= bb; b += 32) cur[b] = start[b] - base;
          __syncwarp();
          scan([&](uint32_t v, uint32_t p) {
            const int b = kf(v);
            if (b >= ba && b <= bb) {
              const int slot = atomicAdd(&cur[b], 1);
              cval[slot] = (T)v;
              cpos[slot] = (uint16_t)p;
            }
          });
        }
        __syncwarp();
        RANK_T(2);
        // buckets up to kLaneSort entries: one bucket per lane, Shell sort
        // (Ciura gaps below the bucket size, ending with an insertion pass)
        // -- smooth data fills many buckets with ~100 candidates, which a
        // warp-wide network would sort one after the other (measured: +15..22 %
        // on smooth fields, +2..6 % on random data)
        constexpr int kLaneSort = 256;
        for (int b = ba + lane; b <= bb; b += 32) {
          const int i0 = start[b] - base, i1 = start[b + 1] - base;
          const int n = i1 - i0;
          if (n > kLaneSort) continue;
          constexpr int kGaps[6] = {132, 57, 23, 10, 4, 1};
#pragma unroll
          for (int gi = 0; gi < 6; gi++) {
            const int gap = kGaps[gi];
            if (gap >= n) continue;
            for (int i = i0 + gap; i < i1; i++) {
              const T v = cval[i];
              const uint16_t p = cpos[i];
              int j = i - gap;
              while (j >= i0 && cval[j] > v) {
                cval[j + gap] = cval[j];
                cpos[j + gap] = cpos[j];
                j -= gap;
              }
              cval[j + gap] = v;
              cpos[j + gap] = p;
            }
          }
        }
        __syncwarp();
        // larger buckets: the warp's bitonic sort, all comparators ascending
        // (mirror stage + half-cleaners), so indices >= n are never touched
        for (int b = ba; b <= bb; b++) {
          const int i0 = start[b] - base, n = start[b + 1] - start[b];
          if (n <= kLaneSort) continue;
          T* a = cval + i0;
          uint16_t* ap = cpos + i0;
          int N = 1;
          while (N < n) N <<= 1;
          auto cmpswap = [&](int lo_i, int hi_i) {
            if (hi_i < n) {
              const T x = a[lo_i], y = a[hi_i];
              if (x > y) {
                const uint16_t px = ap[lo_i];
                a[lo_i] = y;
                a[hi_i] = x;
                ap[lo_i] = ap[hi_i];
                ap[hi_i] = px;
              }
            }
          };
          for (int kk = 2; kk <= N; kk <<= 1) {
            const int hk = kk >> 1;
            for (int i = lane; i < N / 2; i += 32) {
              const int blk = (i / hk) * kk, o = i % hk;
              cmpswap(blk + o, blk + kk - 1 - o);
            }
            __syncwarp();
            for (int j = hk >> 1; j > 0; j >>= 1) {
              for (int i = lane; i < N / 2; i += 32) {
                const int l = 2 * j * (i / j) + (i % j);
                cmpswap(l, l + j);
              }
              __syncwarp();
            }
          }
        }
        __syncwarp();
        RANK_T(3);
        sweep(kf, [&](int t) {
#pragma unroll
          for (int c = 0; c < 2; c++) {
            const int b = sw.m[c];
            if (b >= ba && b <= bb) {
              // r'-th in-window candidate of bucket b, in sorted order
              int need = sw.r2 - sw.bl[c];
              uint32_t v = 0;
              const int cx = 2 * lane + c;  // window columns [cx, cx + K), rows [t, t + K)
              // 4 candidates per round (independent loads), then the exact hit
              const uint32_t pbase = ((uint32_t)t << 8) | (uint32_t)cx;
              auto inwin = [&](uint32_t p) -> int {
                const uint32_t d = p - pbase;  // column offset in bits 0..7 (row checked apart)
                return (d & 0xFFu) < (uint32_t)K && ((p >> 8) - (uint32_t)t) < (uint32_t)KH;
              };
              int i = start[b] - base;
              const int i1 = start[b + 1] - base;
              for (; i + 4 <= i1; i += 4) {
                const int w0 = inwin(cpos[i]), w1 = inwin(cpos[i + 1]), w2 = inwin(cpos[i + 2]),
                          w3 = inwin(cpos[i + 3]);
                const int n4 = w0 + w1 + w2 + w3;
                if (n4 >= need) {
                  const int j = need <= w0 ? 0 : need <= w0 + w1 ? 1 : need <= w0 + w1 + w2 ? 2 : 3;
                  v = cval[i + j];
                  need = 0;
                  break;
                }
                need -= n4;
              }
              for (; need > 0 && i < i1; i++)
                if (inwin(cpos[i]) && --need == 0) v = cval[i];
              put(t, c, v);
            }
          }
        });
      };

      int sp = 0;  // interval stack depth (warp-uniform); entries (lo, hi, bin width)
      auto push = [&](uint32_t a, uint32_t b, uint32_t w) {
        if (lane == 0) {
          stk[3 * sp] = a;
          stk[3 * sp + 1] = b;
          stk[3 * sp + 2] = w;
        }
        sp++;
        __syncwarp();
      };
      // ---- 0. guess the value range from every 8th footprint row -----------
      uint32_t gmin = 0xFFFFFFFFu, gmax = 0u;
      scan_rows(8, [&](uint32_t v, uint32_t) {
        gmin = min(gmin, v);
        gmax = max(gmax, v);
      });
      gmin = warp_min(gmin);
      gmax = warp_max(gmax);
      // ---- 1. first sweep over the guess; the stash measures the true range --
      // keys are monotone in v, so a pixel's bin still brackets its median when
      // samples fall outside the guess (they clamp to bins 0 / NB-1, whose
      // value ranges end at the true footprint extremes)
      if (gmax - gmin < kInner) {
        // at most 126 values guessed: one value per bin -- pixels whose median
        // lies inside are final; the clamped ends become intervals
        const KeyFn<NB, 0> kx{gmin, gmax, 0u, 0};
        int lo_any = 0, hi_any = 0;
        sweep(kx, [&](int t) {
#pragma unroll
          for (int c = 0; c < 2; c++) {
            const int bb = sw.m[c];
            if (bb >= 1 && bb <= NB - 2) put(t, c, gmin + (uint32_t)(bb - 1));
            if (x + c < W) {
              lo_any |= bb == 0;
              hi_any |= bb == NB - 1;
            }
          }
        }, true);
        fmin = warp_min(fmin);
        fmax = warp_max(fmax);
        if (__any_sync(0xffffffffu, lo_any) && fmin < gmin) push(fmin, gmin - 1, gmin - fmin);
        if (__any_sync(0xffffffffu, hi_any) && fmax > gmax) push(gmax + 1, fmax, fmax - gmax);
      } else {
        const int s = 25 - __clz(gmax - gmin);  // bit length - 7 (>= 0: the range is >= 126)
        int blo = NB - 1, bhi = 0;
        sweep(KeyFn<NB, -1>{gmin, gmax, 0u, s}, [&](int) {
          if (x < W) {
            blo = min(blo, sw.m[0]);
            bhi = max(bhi, sw.m[0]);
          }
          if (x + 1 < W) {
            blo = min(blo, sw.m[1]);
            bhi = max(bhi, sw.m[1]);
          }
        }, true);
        blo = (int)warp_min((uint32_t)blo);
        bhi = (int)warp_max((uint32_t)bhi);
        fmin = warp_min(fmin);
        fmax = warp_max(fmax);
        const uint32_t lo = blo == 0 ? fmin : gmin + ((uint32_t)blo << s);
        const uint32_t hi = bhi == NB - 1
                                ? fmax
                                : (uint32_t)min((uint64_t)fmax, (uint64_t)gmin + (((uint64_t)bhi + 1) << s) - 1);
        push(max(lo, fmin), hi, 1u << s);
      }
      RANK_T(0);
      // ---- 2. resolve every interval that may hold medians ------------------
      while (sp > 0) {
        sp--;
        uint32_t lo = stk[3 * sp], hi = stk[3 * sp + 1];
        const uint32_t wprev = stk[3 * sp + 2];  // width of the bins that produced it
        __syncwarp();
        const uint64_t span = (uint64_t)(hi - lo) + 1;
        if (span <= kInner) {
          slice(lo, hi);
          continue;
        }
        // count scan: candidates (samples in [lo, hi]) per fine bucket with
        // lane-private counters in the (idle) histogram words -- counter
        // (bucket, lane) at word bucket * 32 + lane, no contention -- plus
        // their exact value range
        const uint32_t mul = (uint32_t)(((uint64_t)kInner << 32) / span);
        const KeyFn<NB, 1> kf{lo, hi, mul, 0};
        uint32_t* lc = smem;
        for (int b = 0; b < NB; b++) lc[b * 32 + lane] = 0;
        __syncwarp();
        uint32_t tmin = 0xFFFFFFFFu, tmax = 0u;
        scan([&](uint32_t v, uint32_t) {
          if (v >= lo && v <= hi) {
            lc[kf(v) * 32 + lane]++;
            tmin = min(tmin, v);
            tmax = max(tmax, v);
          }
        });
        __syncwarp();
        int n_cand;
        {
          int run = 0;  // bucket offsets start[b]: prefix over buckets (warp-uniform)
          for (int b0 = 0; b0 < NB; b0 += 32) {
            uint32_t c = 0;  // bucket b0 + lane, summed over the lanes' counters
#pragma unroll 8
            for (int l = 0; l < 32; l++) c += lc[(b0 + lane) * 32 + ((l + lane) & 31)];
            int incl = (int)c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += y;
            }
            start[b0 + lane] = run + incl - (int)c;
            run += __shfl_sync(0xffffffffu, incl, 31);
          }
          n_cand = run;
          if (lane == 0) start[NB] = n_cand;
        }
        __syncwarp();
        RANK_T(1);
        if (n_cand == 0) continue;
        if (n_cand <= C::CMAX) {
          resolve(kf, 1, NB - 2);
          continue;
        }
        // too many candidates: the medians are spread (gradients, smooth
        // fields, impulse noise over them)
        lo = warp_min(tmin);
        hi = warp_max(tmax);
        const uint64_t span2 = (uint64_t)(hi - lo) + 1;
        const uint64_t wnew = (span2 + kInner - 1) / kInner;  // bucket width over [lo, hi]
        const int nsl = (int)min((uint64_t)1 << 20, wnew);     // exact slices to cover it
        const int ngr = (n_cand + (C::CMAX * 3 / 4) - 1) / (C::CMAX * 3 / 4);
        if (nsl <= 2 || nsl <= ngr) {  // few values: exact slices
          slices(lo, hi);
          continue;
        }
        if ((uint64_t)wprev >= 4 * wnew && sp < kStack) {
          // the candidates reach far beyond the medians (outliers, gaps):
          // an interval sweep of 126 buckets over [lo, hi], then the samples
          // of the buckets holding medians give the next interval
          const KeyFn<NB, 1> km{lo, hi, (uint32_t)(((uint64_t)kInner << 32) / span2), 0};
          int b0, b1;
          range_pass(km, b0, b1);
          if (b0 > b1) continue;  // no median inside [lo, hi]
          uint32_t t0 = 0xFFFFFFFFu, t1 = 0u;
          scan([&](uint32_t v, uint32_t) {
            const int kb = km(v);
            if (kb >= b0 && kb <= b1) {
              t0 = min(t0, v);
              t1 = max(t1, v);
            }
          });
          push(warp_min(t0), warp_max(t1), (uint32_t)wnew);
          continue;
        }
        // dense spread candidates: groups of consecutive buckets that fit,
        // one fine sweep each.  With a global staging area every candidate is
        // placed once (one footprint scan) and each group copies its
        // contiguous bucket range into shared memory, instead of one
        // placement scan of the whole footprint per group.
        const bool staged = gval != nullptr;
        if (staged) {
          for (int b = lane; b < NB; b += 32) cur[b] = start[b];
          __syncwarp();
          scan([&](uint32_t v, uint32_t p) {
            const int b = kf(v);
            if (b >= 1 && b <= NB - 2) {
              const int slot = atomicAdd(&cur[b], 1);
              gval[slot] = (T)v;
              gpos[slot] = (uint16_t)p;
            }
          });
          __syncwarp();
        }
        for (int b = 1; b <= NB - 2;) {
          const int cb = start[b + 1] - start[b];
          if (cb > C::CMAX) {
            // one bucket alone does not fit: its exact value range becomes an
            // interval of its own (126 finer buckets), or slices if the stack is full
            const uint32_t v0 = kf.first_of(b), v1 = kf.first_of(b + 1) - 1;
            if (sp < kStack)
              push(v0, v1, (uint32_t)min((uint64_t)0xFFFFFFFFu, (span + kInner - 1) / kInner));
            else
              slices(v0, v1);
            b++;
            continue;
          }
          int e = b;
          while (e + 1 <= NB - 2 && start[e + 2] - start[b] <= C::CMAX) e++;
          if (start[e + 1] > start[b]) resolve(kf, b, e, staged);
          b = e + 1;
        }
      }
      RANK_T(4);
    }
  }
}

// Square K x K (RT = false, kh = K) or rectangular K x kh (RT = true).
template <typename T, int K, bool RT = false>
int launch_rank_k(const Job& job, cudaStream_t stream, int kh = K) {
  using C = RankCfg<T, K>;
  static_assert(C::kWarpBytes <= 227 * 1024, "rank kernel does not fit in shared memory");
  const int kSmem = RT ? C::kWarpBytes - C::kRingBytes +
                             (((kh + 2 * C::G + 1) * C::KW + 15) / 16) * 16
                       : C::kWarpBytes;
  auto fn = rank_kernel<T, K, RT>;
  LaunchInfo li;
  if (!RT) {
    static LaunchCache cache;
    li = cache.get(fn, 32, kSmem);
  } else {  // the ring (and so the occupancy) depends on kh
    li = launch_info(fn, 32, kSmem);
  }
  if (li.err != cudaSuccess) return (int)li.err;
  const int sms = li.sms, occ = li.occ;
  const int n_strips = (job.width + 63) / 64;
  const long slots = (long)sms * occ;
  // every segment count with R = ceil(out_h / segs) <= RMAX, so the item
  // count can land just under a multiple of the resident warps
  int best_R = C::RMAX;
  long best_cost = 0x7fffffffffffL;
  for (int segs = (job.out_h + C::RMAX - 1) / C::RMAX; segs <= (job.out_h + 7) / 8; segs++) {
    const int R = (job.out_h + segs - 1) / segs;
    const long items = (long)segs * n_strips * job.channels;
    const long waves = (items + slots - 1) / slots;
    // two sweeps of (rows + ~K build) each
    const long cost = waves * (long)(R + kh + 8);
    if (cost < best_cost) {
      best_cost = cost;
      best_R = R;
    }
  }
  const int R = best_R;
  const int n_segs = (job.out_h + R - 1) / R;
  const long items = (long)n_segs * n_strips * job.channels;
  const int grid = (int)(items < slots ? items : slots);
  // global staging for spread candidates: one footprint's worth per resident
  // warp, stream-ordered from a private pool (kernel falls back to one
  // placement scan per group when the allocation fails)
  const int gcap = C::FW * (R + kh - 1);
  const int64_t gstride = (((int64_t)gcap * (int64_t)(sizeof(T) + 2)) + 255) / 256 * 256;
  uint8_t* gstage = static_cast<uint8_t*>(rank_stage_alloc((size_t)gstride * grid, stream));
  fn<<<grid, 32, kSmem, stream>>>(job, R, n_strips, n_segs, kh, gstage, gstride, gcap);
  const int err = (int)cudaGetLastError();
  if (gstage) rank_stage_free(gstage, stream);
  return err;
}

}  // namespace
}  // namespace tmb
