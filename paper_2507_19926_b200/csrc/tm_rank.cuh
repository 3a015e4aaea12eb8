// tm_rank.cuh -- data-aware O(k) median for 16- and 32-bit images (variant (2)
// for uint16 / uint32): the sliding-histogram sweep (tm_sweep.cuh) run twice
// on 7-bit KEYS derived from the samples.
//
// Reference role: the data-aware engine (aware.py:437-492) -- the candidates
// for a tile of outputs are narrowed with a cheap pass, then the median is
// selected exactly by rank among the survivors (the paper's forgetful
// candidate windows, section 5.1, applied per tile of outputs).
//
// One warp = one work item: 64 output columns x up to RMAX output rows.
//  1. coarse pass: sweep with key = the top 7 bits of each sample.  Gives every
//     output pixel the exact 7-bit prefix of its median; every median of the
//     item lies in [lo, hi] = [B_lo << s, ((B_hi + 1) << s) - 1].
//  2. fine keys: 0 below lo, 127 above hi, 1 + floor((v - lo) * 125 / span)
//     inside (value-width bins, monotone in v, computed from the value alone;
//     one value per bin when the span is at most 125).  When bins hold several
//     values the
//     candidates (samples in [lo, hi]) are bucketed by key (count, exclusive
//     scan, place) and each bucket is sorted by value, so bin b's candidates
//     are the sorted range [start[b], start[b+1]).
//  3. fine pass: sweep over the fine keys.  The walk lands every pixel in a bin
//     b with residual rank r' = R2 - #keys < b; the median is lo + b - 1 for
//     one-value bins, else the r'-th candidate of bin b (in sorted order) inside the
//     pixel's window.
// Exact by construction.  If an item has more candidates than fit (CMAX) it
// is split in halves by rows (down to single rows); a row that still does not
// fit is selected per pixel by brute force (radix selection over the window)
// -- only adversarial high-entropy data gets there.
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
#ifndef TMB_RANK_FINE_BINS
#define TMB_RANK_FINE_BINS 128
#endif
  static constexpr int NBC = 128;                      // coarse key bins (top 7 bits)
  static constexpr int NB = TMB_RANK_FINE_BINS;        // fine key bins
  using SWC = WarpSweep<K, NBC>;
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
  static constexpr int kStartBytes = (NB + 16) * 4;      // start[]
  static constexpr int kHistBytes = SW::kHistBytes > SWC::kHistBytes ? SW::kHistBytes : SWC::kHistBytes;
  static constexpr int kWarpBytes = kHistBytes + kRingBytes + kValBytes + kPosBytes + kStartBytes;
  static constexpr int BITS = 8 * (int)sizeof(T);
  static constexpr int SHIFT = BITS - 7;               // coarse key = top 7 bits (NBC)
  static constexpr int E = (G * FW + 31) / 32;         // prefetch samples per lane
};

template <typename T>
__device__ __forceinline__ uint32_t load_s(const T* src, const Job& job, int y, int x) {
  return __ldg(src + (int64_t)y * job.src_pitch + (int64_t)x * job.channels);
}

// Brute-force exact median of one pixel (last-resort path): MSB-first radix
// selection over the clamped window, one bit per pass.
template <typename T, int K>
__device__ uint32_t brute_median(const T* src, const Job& job, int yc, int xc) {
  constexpr int R2 = (K * K + 1) / 2;
  uint32_t prefix = 0, need = R2;
  for (int bit = 8 * (int)sizeof(T) - 1; bit >= 0; bit--) {
    const uint32_t hi_mask = bit + 1 >= 32 ? 0u : (~0u << (bit + 1));
    uint32_t zeros = 0;
    for (int dy = -K / 2; dy <= K / 2; dy++) {
      const int y = clampi(yc + dy, 0, job.src_h - 1);
      for (int dx = -K / 2; dx <= K / 2; dx++) {
        const uint32_t v = load_s(src, job, y, clampi(xc + dx, 0, job.width - 1));
        zeros += ((v & hi_mask) == prefix) && !((v >> bit) & 1u);
      }
    }
    if (need > zeros) {
      need -= zeros;
      prefix |= 1u << bit;
    }
  }
  return prefix;
}

// Key of a sample: coarse pass (f < 0): top 7 bits; fine pass: 0 / NB-1 outside
// [lo, hi], 1 + floor((v - lo) * (NB - 2) / span) inside.
template <int NB>
struct KeyFn {
  uint32_t lo, hi;
  uint32_t mul;  // fine: bin = (v - lo) * mul >> 32, all NB - 2 inner bins in use
  int f;         // < 0: coarse; 0: one value per bin; > 0: multi-value bins
  int shift;
  __device__ __forceinline__ uint8_t operator()(uint32_t v) const {
    if (f < 0) return (uint8_t)(v >> shift);
    if (v < lo) return 0;
    if (v > hi) return NB - 1;
    return (uint8_t)(1 + (f == 0 ? v - lo : __umulhi(v - lo, mul)));
  }
};

#ifdef TMB_RANK_PROFILE
static __device__ unsigned long long g_rank_prof[8];  // per translation unit; tm_rank.cu sums them
#define RANK_T(i) do { const long long _n = clock64(); if (lane == 0) atomicAdd(&g_rank_prof[i], (unsigned long long)(_n - _t)); _t = _n; } while (0)
#else
#define RANK_T(i) do { } while (0)
#endif

template <typename T, int K>
__global__ void __launch_bounds__(32) rank_kernel(Job job, int R, int n_strips, int n_segs) {
  using C = RankCfg<T, K>;
  using SW = typename C::SW;
  extern __shared__ __align__(16) uint32_t smem[];
  const int lane = threadIdx.x;
  uint8_t* ring = reinterpret_cast<uint8_t*>(smem) + C::kHistBytes;
  T* cval = reinterpret_cast<T*>(ring + C::kRingBytes);                  // bucketed candidates
  uint16_t* cpos = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(cval) + C::kValBytes);
  int* start = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(cpos) + C::kPosBytes);
  typename C::SWC swc;  // coarse and fine sweeps share the histogram words
  SW sw;
  swc.init(smem, lane);
  sw.init(smem, lane);
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

    int Rcur = rows_item;
    for (int y0 = 0; y0 < rows_item;) {
      const int rows = min(Rcur, rows_item - y0);
      const int Y0 = Yi + y0;
      const int sy_base = job.out_y0 + Y0 - C::H;  // source row of footprint row 0
      const int q_end = K + rows - 1;              // footprint rows

      // G footprint rows of samples [q0, q0 + G) into registers.
      auto fetch_raw = [&](int q0, uint32_t (&v)[C::E]) {
#pragma unroll
        for (int e = 0; e < C::E; e++) {
          const int idx = lane + e * 32;
          const int g = idx / C::FW, c = idx - (idx / C::FW) * C::FW;
          v[e] = (idx < C::G * C::FW && q0 + g < q_end)
                     ? load_s(src, job, clampi(sy_base + q0 + g, 0, SH - 1),
                              clampi(X0 - C::H + c, 0, W - 1))
                     : 0u;
        }
      };
      auto valid = [&](int q0, int e) {
        const int idx = lane + e * 32;
        return idx < C::G * C::FW && q0 + idx / C::FW < q_end;
      };
      auto pos_of = [&](int q0, int e) {
        const int idx = lane + e * 32;
        const int g = idx / C::FW, c = idx - (idx / C::FW) * C::FW;
        return (uint32_t)(((q0 + g) << 8) | c);
      };

      // One sweep over the sub-item with keys from `kf`; `emit(t)` after each row.
      auto sweep = [&](auto& sw, const auto& kf, auto&& emit) {
        using S = typename std::remove_reference<decltype(sw)>::type;
        auto stash = [&](int q0, const uint32_t (&v)[C::E]) {
#pragma unroll
          for (int e = 0; e < C::E; e++) {
            const int idx = lane + e * 32;
            const int g = idx / C::FW, c = idx - (idx / C::FW) * C::FW;
            if (valid(q0, e)) ring[((q0 + g) % C::RING) * C::KW + c] = kf(v[e]);
          }
        };
        auto row = [&](int q) { return ring + (q % C::RING) * C::KW; };
        __syncwarp();
        {
          // prologue: rows [0, K + G), loads double-buffered against stores
          uint32_t va[C::E], vb[C::E];
          fetch_raw(0, va);
          int q = 0;
          for (; q + C::G < K + C::G; q += 2 * C::G) {
            fetch_raw(q + C::G, vb);
            stash(q, va);
            if (q + 2 * C::G < K + C::G) fetch_raw(q + 2 * C::G, va);
            stash(q + C::G, vb);
          }
          if (q < K + C::G) stash(q, va);
        }
        sw.zero();
        __syncwarp();
        for (int q = 0; q < K; q++) {
          uint32_t ch[S::NC];
          S::chunks(row(q), lane, ch);
          sw.add_row(ch);
        }
        sw.init_median();
        emit(0);
        for (int t0 = 1; t0 < rows; t0 += C::G) {
          uint32_t nxt[C::E];
          const int qn = K + t0 - 1 + C::G;
          if (qn < q_end) fetch_raw(qn, nxt);
          const int t1 = min(t0 + C::G, rows);
          for (int t = t0; t < t1; t++) {
            uint32_t co[S::NC], ci[S::NC];
            S::chunks(row(t - 1), lane, co);
            S::chunks(row(t - 1 + K), lane, ci);
            sw.step(co, ci);
            emit(t);
          }
          if (qn < q_end) stash(qn, nxt);
          __syncwarp();
        }
      };

#ifdef TMB_RANK_PROFILE
      long long _t = clock64();
#endif
      // ---- 1. candidate range: the exact coarse pass ------------------------
      uint32_t lo, hi;
      {
        int blo = C::NBC - 1, bhi = 0;
        KeyFn<C::NBC> kc{0u, 0u, 0u, -1, C::SHIFT};
        sweep(swc, kc, [&](int) {
          if (x < W) {
            blo = min(blo, swc.m[0]);
            bhi = max(bhi, swc.m[0]);
          }
          if (x + 1 < W) {
            blo = min(blo, swc.m[1]);
            bhi = max(bhi, swc.m[1]);
          }
        });
        for (int o = 16; o; o >>= 1) {
          blo = min(blo, __shfl_xor_sync(0xffffffffu, blo, o));
          bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
        }
        lo = (uint32_t)blo << C::SHIFT;
        hi = (uint32_t)(((uint64_t)(bhi + 1) << C::SHIFT) - 1);
      }
      // value -> fine bin: identity when [lo, hi] has at most NB - 2 values,
      // else floor((v - lo) * (NB - 2) / (hi - lo + 1)) via a 32.32 multiplier
      const uint64_t span = (uint64_t)(hi - lo) + 1;
      const int f = span <= (uint64_t)(C::NB - 2) ? 0 : 1;
      const uint32_t mul = f ? (uint32_t)((((uint64_t)(C::NB - 2)) << 32) / span) : 0u;
      const KeyFn<C::NB> kf{lo, hi, mul, f, 0};

      RANK_T(0);
      // ---- 2. candidates bucketed by fine key (only when f > 0) ----------
      // Two scans of the footprint: count per key, then place each candidate
      // at its bucket's cursor; each bucket is then sorted by value.
      int n_cand = 0;
      if (f > 0) {
        // lane-private bucket counters in the (idle) histogram words:
        // counter (bucket, lane) at word bucket * 32 + lane -- no contention
        uint32_t* lc = smem;
        for (int b = 0; b < C::NB; b++) lc[b * 32 + lane] = 0;
        __syncwarp();
        auto scan = [&](auto&& visit) {
          uint32_t va[C::E], vb[C::E];
          fetch_raw(0, va);
          auto visit_all = [&](int q0, const uint32_t (&v)[C::E]) {
#pragma unroll
            for (int e = 0; e < C::E; e++)
              if (valid(q0, e) && v[e] >= lo && v[e] <= hi) visit(v[e], pos_of(q0, e));
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
        scan([&](uint32_t v, uint32_t) { lc[kf(v) * 32 + lane]++; });
        __syncwarp();
        // exclusive scan over (bucket, lane): bucket b of lane l starts at
        // start[b] + sum of lanes < l; lane l walks the buckets in order
        {
          int run = 0;  // prefix over buckets (warp-uniform)
          for (int b = 0; b < C::NB; b++) {
            const int c = (int)lc[b * 32 + lane];
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += y;
            }
            lc[b * 32 + lane] = (uint32_t)(run + incl - c);  // this lane's cursor
            if (lane == 0) start[b] = run;
            run += __shfl_sync(0xffffffffu, incl, 31);
          }
          n_cand = run;
          if (lane == 0) start[C::NB] = n_cand;
        }
        __syncwarp();
        if (n_cand > C::CMAX) {
          if (rows > 1) {  // too many candidates: halve the sub-item
            Rcur = (rows + 1) / 2;
            continue;
          }
          for (int c = 0; c < 2; c++)  // a single row that still does not fit
            if (x + c < W)
              dst[(int64_t)Y0 * job.dst_pitch + (int64_t)(x + c) * CH] =
                  (T)brute_median<T, K>(src, job, job.out_y0 + Y0, x + c);
          y0 += rows;
          Rcur = rows_item;
          continue;
        }
        RANK_T(1);
        scan([&](uint32_t v, uint32_t p) {
          const int slot = (int)(lc[kf(v) * 32 + lane]++);
          cval[slot] = (T)v;
          cpos[slot] = (uint16_t)p;
        });
        __syncwarp();
        RANK_T(2);
        // sort each bucket by value: insertion sort per lane for small
        // buckets, the whole warp (odd-even transposition) for large ones
        for (int b = 1 + lane; b < C::NB - 1; b += 32) {
          const int i0 = start[b], i1 = start[b + 1];
          if (i1 - i0 > 64) continue;
          for (int i = i0 + 1; i < i1; i++) {
            const T v = cval[i];
            const uint16_t p = cpos[i];
            int j = i - 1;
            while (j >= i0 && cval[j] > v) {
              cval[j + 1] = cval[j];
              cpos[j + 1] = cpos[j];
              j--;
            }
            cval[j + 1] = v;
            cpos[j + 1] = p;
          }
        }
        __syncwarp();
        for (int b = 1; b < C::NB - 1; b++) {
          const int i0 = start[b], n = start[b + 1] - i0;
          if (n <= 64) continue;
          for (int ph = 0; ph < n; ph++) {
            for (int i = i0 + (ph & 1) + 2 * lane; i + 1 < i0 + n; i += 64) {
              const T a = cval[i], c = cval[i + 1];
              if (a > c) {
                const uint16_t pa = cpos[i];
                cval[i] = c;
                cval[i + 1] = a;
                cpos[i] = cpos[i + 1];
                cpos[i + 1] = pa;
              }
            }
            __syncwarp();
          }
        }
      }

      RANK_T(3);
      // ---- 3. fine pass -----------------------------------------------------
      sweep(sw, kf, [&](int t) {
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const int b = sw.m[c];
          uint32_t v = 0;
          if (b < 1 || b > C::NB - 2) {
            // only columns beyond the image edge (excluded from [lo, hi]) land here
          } else if (f == 0) {
            v = lo + (uint32_t)(b - 1);
          } else {
            // r'-th in-window candidate of bin b, in sorted order
            int need = SW::R2 - sw.bl[c];
            const int cx = 2 * lane + c;  // window columns [cx, cx + K), rows [t, t + K)
            // 4 candidates per round (independent loads), then the exact hit
            const uint32_t base = ((uint32_t)t << 8) | (uint32_t)cx;
            auto inwin = [&](uint32_t p) -> int {
              const uint32_t d = p - base;  // column offset in bits 0..7 (row checked apart)
              return (d & 0xFFu) < (uint32_t)K && ((p >> 8) - (uint32_t)t) < (uint32_t)K;
            };
            int i = start[b];
            const int i1 = start[b + 1];
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
          }
          if (x + c < W) dst[(int64_t)(Y0 + t) * job.dst_pitch + (int64_t)(x + c) * CH] = (T)v;
        }
      });
      RANK_T(4);
      y0 += rows;
      Rcur = rows_item;
    }
  }
}

template <typename T, int K>
int launch_rank_k(const Job& job, cudaStream_t stream) {
  using C = RankCfg<T, K>;
  constexpr int kSmem = C::kWarpBytes;
  static_assert(kSmem <= 227 * 1024, "rank kernel does not fit in shared memory");
  auto fn = rank_kernel<T, K>;
  static const LaunchInfo li = launch_info(fn, 32, kSmem);
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
    const long cost = waves * (long)(R + K + 8);
    if (cost < best_cost) {
      best_cost = cost;
      best_R = R;
    }
  }
  const int R = best_R;
  const int n_segs = (job.out_h + R - 1) / R;
  const long items = (long)n_segs * n_strips * job.channels;
  const int grid = (int)(items < slots ? items : slots);
  fn<<<grid, 32, kSmem, stream>>>(job, R, n_strips, n_segs);
  return (int)cudaGetLastError();
}

}  // namespace
}  // namespace tmb
