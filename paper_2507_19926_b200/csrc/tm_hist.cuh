// tm_hist.cuh -- data-aware O(k) median for 8-bit images: sliding column
// histograms swept down the image (variant (2) for uint8).  Square kernels
// are instantiated in tm_hist.cu, rectangular k_w x k_h ones in
// tm_hist_rect.cu (window width a template parameter, height at run time).
//
// Reference role: the data-aware engine (aware.py:437-492, section 5)
// shares sorted runs between neighbouring output pixels so the work per pixel
// grows O(k) instead of O(k^2).  For 8-bit samples the cheapest shareable
// structure on a GPU is the window histogram itself: moving the window one row
// down removes k_w samples and adds k_w samples, and the median -- rank
// r = (k_w k_h + 1)/2 of the clamped window (geometry.py:55-58,
// reference.py:26-43) -- is found by walking from the previous median, which
// moves little from row to row.  Exact by construction: the histogram is the
// window multiset.
//
// One warp = one work item: 32 x CPL adjacent output columns x a run of output
// rows of one channel (tm_sweep.cuh: CPL columns per lane share one count word
// per bin, one shared-memory RED per sample and row step serves them all; the
// packed walk moves every column's median together).  The ring holds the last
// k_h + 2G + 1 footprint rows (clamped reads = replicate borders), refilled G
// rows at a time from registers prefetched a group ahead.  Long images give
// every resident warp one equal piece of the columns' rows laid end to end;
// short ones are cut into the segment count with the smallest makespan.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tm_common.cuh"
#include "tm_kernels.h"
#include "tm_sweep.cuh"

namespace tmb {
namespace {

// K = window width (template), window height K (square) or a runtime kh.
// CPLV = output columns per lane: 3 (10-bit count fields, K x kh < 512) or 2.
template <int K, int G, int CPLV>
struct HistCfg {
  using S = WarpSweep<K, 256, CPLV>;
  static constexpr int CPL = S::kCPL;
  static constexpr int H = K / 2;                   // horizontal halo
  static constexpr int RING = K + 2 * G + 1;        // square: next group lands while this one runs
  static constexpr int FW = S::COLS + K - 1;        // footprint columns of the warp
  // ring row bytes: the last lane's chunk words end at ((CPL*31)/4 + NC + 1) words
  // (measured per-byte: every byte of the smem budget counts -- 6 warps/SM need
  // <= 37888 B per 1-warp CTA)
  static constexpr int RW0 = ((FW + 3) / 4) * 4;
  static constexpr int RWL = ((S::kCPL * 31) / 4 + S::NWD) * 4;
  static constexpr int RW = RW0 > RWL ? RW0 : RWL;
  static constexpr int kRingBytes = RING * RW;
  static constexpr int kWarpBytes = S::kHistBytes + kRingBytes;
  static constexpr int E = (G * FW + 31) / 32;      // prefetch bytes per lane
};

// One warp per work item (32*CPL output columns x R rows of one channel); the
// warps of a CTA share nothing, so there is no CTA barrier anywhere.  RT: the
// window height is the runtime `kh_rt` (rectangular K x kh kernels), else K.
template <int K, int G, int WPC, int CPLV, bool RT>
__global__ void __launch_bounds__(32 * WPC)
    hist8_kernel(Job job, int R, int n_strips, int n_segs, int kh_rt) {
  using C = HistCfg<K, G, CPLV>;
  using SW = typename C::S;
  extern __shared__ __align__(16) uint32_t smem[];
  const int KH = RT ? kh_rt : K;                   // window height
  const int HH = KH / 2;                           // vertical halo
  const int RING = RT ? KH + 2 * G + 1 : C::RING;  // ring rows
  const int warp = threadIdx.x >> 5;
  const int tid = threadIdx.x & 31;
  uint32_t* wbase = smem + warp * ((SW::kHistBytes + RING * C::RW) / 4);
  uint8_t* ring = reinterpret_cast<uint8_t*>(wbase) + SW::kHistBytes;
  SW sw;
  sw.init(wbase, tid, (K * KH + 1) / 2);
  const int W = job.width, SH = job.src_h, CH = job.channels;
  const int n_items = n_strips * CH * n_segs;

  // Work assignment.  n_segs > 0: items of R rows (segment s of a column
  // strip), grid-stride.  n_segs < 0: continuous mode with blocks of
  // nsg = -n_segs adjacent strips -- the blocks' output rows laid end to end
  // and cut into one equal piece per group of nsg x CH consecutive warps, the
  // group's warps filtering (strip in block, channel) of the same rows side
  // by side: every warp does the same row count (a piece crossing a block
  // boundary runs as two sub-items), so no SM idles at the end, and the halo
  // columns of neighbouring strips and the channels of interleaved rows are
  // read from L2 by concurrent warps (each line leaves DRAM about once, output
  // sectors fill in L2 before write-back).
  const int gw = blockIdx.x * WPC + warp;
  int item = gw;
  int sub_strip = 0, sub_chan = 0, nsg = 1;
  int64_t p0 = 0, p1 = 0;
  if (n_segs < 0) {
    nsg = -n_segs;
    const int gsize = nsg * CH;
    const int groups = gridDim.x * WPC / gsize;  // the last < gsize warps idle
    const int grp = gw / gsize;
    const int sub = gw - grp * gsize;
    sub_chan = sub % CH;
    sub_strip = sub / CH;
    if (grp < groups) {
      const int64_t total = (int64_t)((n_strips + nsg - 1) / nsg) * job.out_h;
      p0 = total * grp / groups;
      p1 = total * (grp + 1) / groups;
    }
  }
  for (;;) {
    int chan, strip, Y0, rows;
    if (n_segs < 0) {
      if (p0 >= p1) break;
      const int64_t bi = p0 / job.out_h;
      Y0 = (int)(p0 - bi * job.out_h);
      rows = (int)min((int64_t)(job.out_h - Y0), p1 - p0);
      chan = sub_chan;
      strip = (int)bi * nsg + sub_strip;
      p0 += rows;
      if (strip >= n_strips) continue;  // the last block is partial
    } else {
      if (item >= n_items) break;
      chan = item % CH;
      strip = (item / CH) % n_strips;
      Y0 = (item / (CH * n_strips)) * R;
      rows = min(R, job.out_h - Y0);
      item += gridDim.x * WPC;
    }
    const int X0 = strip * SW::COLS;
    const uint8_t* src = static_cast<const uint8_t*>(job.src) + chan;
    uint8_t* dst = static_cast<uint8_t*>(job.dst) + chan;
    const int sy_base = job.out_y0 + Y0 - HH;    // source row of ring row q = 0
    const int q_end = KH + rows - 1;             // ring rows of this item: [0, q_end)

    // Slot e of a lane fetches group row g_e, footprint column c_e; both and
    // the clamped column offset are fixed per item (computed once here), so a
    // fetch costs a row clamp, one wide multiply-add and the load.
    int g_of[C::E], xo[C::E], ro[C::E];
#pragma unroll
    for (int e = 0; e < C::E; e++) {
      const int idx = tid + e * 32;
      const int g = idx / C::FW, c = idx - g * C::FW;
      g_of[e] = idx < G * C::FW ? g : 0x3fffffff;  // an unused slot never passes q < q_end
      xo[e] = clampi(X0 - C::H + c, 0, W - 1) * CH;
      ro[e] = g * C::RW + c;                       // byte of the slot in its ring row
    }
    auto fetch = [&](int q0, uint8_t (&v)[C::E]) {
#pragma unroll
      for (int e = 0; e < C::E; e++) {
        if (q0 + g_of[e] < q_end) {
          const int sy = clampi(sy_base + q0 + g_of[e], 0, SH - 1);
          v[e] = __ldg(src + (int64_t)sy * job.src_pitch + xo[e]);
        }
      }
    };
    auto stash = [&](int q0, const uint8_t (&v)[C::E]) {
      // ring rows q0 .. q0 + G - 1 are consecutive modulo RING: one base
      const int r0 = q0 % RING;
      uint8_t* rb = ring + r0 * C::RW;
#pragma unroll
      for (int e = 0; e < C::E; e++) {
        if (q0 + g_of[e] < q_end) {
          const int r = r0 + g_of[e];
          rb[ro[e] - (r >= RING ? RING * C::RW : 0)] = v[e];
        }
      }
    };
    auto row = [&](int q) { return ring + (q % RING) * C::RW; };

    __syncwarp();  // previous item of this warp done with the ring
    for (int q = 0; q < KH + G; q += G) {
      uint8_t v[C::E];
      fetch(q, v);
      stash(q, v);
    }
    sw.zero();
    __syncwarp();

    // ---- build the first window: rows q = 0 .. KH-1 -----------------------
    for (int q = 0; q < KH; q++) {
      uint32_t ch[SW::NC];
      SW::chunks(row(q), tid, ch);
      sw.add_row(ch);
    }
    sw.init_median();
    const int x = X0 + C::CPL * tid;
    // output pointer advanced one row per store; column predicates fixed per item
    uint8_t* dp = dst + (int64_t)Y0 * job.dst_pitch + (int64_t)x * CH;
    const int64_t dpitch = job.dst_pitch;
    bool col_ok[C::CPL];
#pragma unroll
    for (int c = 0; c < C::CPL; c++) col_ok[c] = x + c < W;
    auto store = [&]() {
#pragma unroll
      for (int c = 0; c < C::CPL; c++)
        if (col_ok[c]) dp[c * CH] = (uint8_t)sw.m[c];
      dp += dpitch;
    };
    store();

    // ---- sweep down: groups of G output rows --------------------------------
    // ring rows of the leaving (t - 1) and entering (t - 1 + KH) footprint
    // rows, advanced one row per step with a wrap (no modulo per step)
    const uint8_t* ring_end = ring + RING * C::RW;
    const uint8_t* po = row(0);
    const uint8_t* pi = row(KH);
    for (int t0 = 1; t0 < rows; t0 += G) {
      uint8_t nxt[C::E];
      const int qn = KH + t0 - 1 + G;  // first ring row of the next group
      if (qn < q_end) fetch(qn, nxt);
      const int t1 = min(t0 + G, rows);
      for (int t = t0; t < t1; t++) {
        uint32_t co[SW::NC], ci[SW::NC];
        SW::chunks(po, tid, co);
        SW::chunks(pi, tid, ci);
        po += C::RW;
        pi += C::RW;
        if (po == ring_end) po = ring;
        if (pi == ring_end) pi = ring;
        sw.step(co, ci);
        store();
      }
      if (qn < q_end) stash(qn, nxt);
      __syncwarp();
    }
  }
}

// Warps per CTA: 1 (CTAs are independent anyway; the hardware packs as many
// as shared memory allows onto each SM).
template <int K>
constexpr int hist_g() {
#ifdef TMB_HIST_G
  return TMB_HIST_G;
#else
  // ring refill group: measured per k range with 2 columns per lane (k = 19, 21:
  // G 8 -> 4 is +14 %; k = 25: G 8 -> 2 is +18 %; k >= 33 prefers 4); 4 for the
  // 3-column lanes (k <= 21) keeps the ring small enough for 6 warps per SM
  return K <= 21 ? 4 : (K <= 31 ? 2 : 4);
#endif
}

// Square K x K (RT = false, kh = K) or rectangular K x kh (RT = true).
template <int K, int CPLV, bool RT>
int launch_hist8_t(const Job& job, int kh, cudaStream_t stream) {
  constexpr int G = hist_g<K>(), WPC = 1;
  using C = HistCfg<K, G, CPLV>;
  const int ring_rows = RT ? kh + 2 * G + 1 : C::RING;
  const int kSmem = (C::S::kHistBytes + ring_rows * C::RW) * WPC;
  static_assert(C::kWarpBytes <= 227 * 1024, "histogram kernel does not fit in shared memory");
  auto fn = hist8_kernel<K, G, WPC, CPLV, RT>;
  LaunchInfo li;
  if (!RT) {
    static LaunchCache cache;
    li = cache.get(fn, 32 * WPC, kSmem);
  } else {  // the ring (and so the occupancy) depends on kh
    li = launch_info(fn, 32 * WPC, kSmem);
  }
  if (li.err != cudaSuccess) return (int)li.err;
  const int sms = li.sms, occ = li.occ;
  const int n_strips = (job.width + C::S::COLS - 1) / C::S::COLS;
  const long slots = (long)sms * occ * WPC;  // concurrent warps
  // Row segment length: long enough to amortise the k x k build (about k rows
  // of work), short enough that the last wave is small -- the candidate with
  // the smallest estimated makespan.
  // every segment count (R = ceil(out_h / segs)), so the item count can land
  // just under a multiple of the resident warps
  int best_R = job.out_h;
  long best_cost = 0x7fffffffffffL;
  for (int segs = 1; segs <= (job.out_h + 15) / 16; segs++) {
    const int R = (job.out_h + segs - 1) / segs;
    if (segs > 1 && R == (job.out_h + segs - 2) / (segs - 1)) continue;  // same R as segs - 1
    const long items = (long)segs * n_strips * job.channels;
    const long waves = (items + slots - 1) / slots;
    const long cost = waves * (long)(R + kh + 8);
    if (cost < best_cost) {
      best_cost = cost;
      best_R = R;
    }
  }
  const int R = best_R;
  int n_segs = (job.out_h + R - 1) / R;
  const long items = (long)n_segs * n_strips * job.channels;
  const long ctas = (items + WPC - 1) / WPC;
  int grid = (int)(ctas < slots / WPC ? ctas : slots / WPC);
#ifndef TMB_HIST_SEGMENTS
  // long pieces: one equal piece per resident warp (continuous mode) beats the
  // best segment count whenever a piece is much longer than the k-row build
  // it may pay twice (C2: 840 segments on 888 warps -> 888 pieces, +3..5 %)
  // groups of nsg adjacent strips x CH channels (about 8 warps)
  const int nsg = std::max(1, std::min(n_strips, 8 / std::max(1, job.channels)));
  const long gsize = (long)nsg * job.channels;
  const long groups = slots / gsize;
  const int64_t blocks = (n_strips + nsg - 1) / nsg;
  const int64_t piece = groups > 0 ? blocks * job.out_h / groups : 0;
  const int64_t builds = piece / job.out_h + 2;  // sub-items a piece may span
  if (groups > 0 && piece >= 4 * (kh + 8) && piece + builds * (kh + 8) < best_cost) {
    n_segs = -nsg;
    grid = (int)(slots / WPC);
  }
#endif
  fn<<<grid, 32 * WPC, kSmem, stream>>>(job, R, n_strips, n_segs, kh);
  return (int)cudaGetLastError();
}

}  // namespace
}  // namespace tmb
