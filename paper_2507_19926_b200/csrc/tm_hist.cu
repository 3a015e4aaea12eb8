// tm_hist.cu -- data-aware O(k) median for 8-bit images: sliding column
// histograms swept down the image (variant (2) for uint8).
//
// Reference role: the data-aware engine (aware.py:437-492, section 5)
// shares sorted runs between neighbouring output pixels so the work per pixel
// grows O(k) instead of O(k^2).  For 8-bit samples the cheapest shareable
// structure on a GPU is the window histogram itself: moving the k x k window
// one row down removes k samples and adds k samples, and the median -- rank
// r = (k^2+1)/2 of the clamped window (geometry.py:55-58, reference.py:26-43)
// -- is found by walking from the previous median, which moves little from
// row to row.  Exact by construction: the histogram is the window multiset.
//
// Work decomposition: one CTA = 2*NT adjacent output columns x a segment of R
// output rows of one channel; a grid-stride loop over (row segment, column
// strip, channel) work items keeps every SM busy to the last item.
//
// Per thread: TWO adjacent output columns (x, x+1) whose histograms share
// storage -- bin v of column x is the low half-word, of column x+1 the high
// half-word of one 32-bit word.  A sample at window column j (0..k relative
// to x) belongs to column x's window when j < k and to x+1's when j > 0, so
// its update is ONE shared-memory atomic add of the compile-time constant
// 0x1 / 0x10001 / 0x10000 (RED.ADD: no return, no read-modify-write round
// trip); k+1 atomics per row step serve two output pixels.  Counts are at most
// k^2 <= 5625 < 2^16 and never negative, so the halves never carry into each
// other.
//
// Shared memory:
//   * hist: bins -4 .. 259 (4 zero bins either side for the 4-bin walk) x NT
//     words, word (bin, thread) at bin * NT + tid: a warp's accesses hit 32
//     distinct banks whatever the bins;
//   * ring: the last k + 2G + 1 source rows of the strip footprint (2*NT + k - 1
//     samples each, clamped reads = replicate borders), refilled G rows at a
//     time from registers prefetched one group ahead.
// `below` (#samples < m) is kept incrementally with SIMD byte compares
// (__vsetltu4 on 4 samples at once); the walk moves m up to 4 bins per round
// trip and is warp-convergent (a converged lane's step is idempotent, so the
// lanes simply loop until all agree).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tm_common.cuh"
#include "tm_kernels.h"

namespace tmb {
namespace {

template <int K, int G>
struct HistCfg {
  static constexpr int NT = 32;                     // one warp = one work item
  static constexpr int H = K / 2;
  static constexpr int RING = K + 2 * G + 1;        // next group lands while this one runs
  static constexpr int FW = 2 * NT + K - 1;         // footprint columns of the warp
  static constexpr int RW = ((FW + 3) / 4) * 4 + 8; // ring row bytes (+ slack words)
  static constexpr int NS = K + 1;                  // window samples per thread per row
  static constexpr int NC = (NS + 3) / 4;           // 4-sample chunks
  static constexpr int NWD = NC + 1;                // aligned words covering the chunks
  static constexpr int kPad = 8;                    // zero bins below 0 / above 255
  static constexpr int kWords = 256 + 2 * kPad;
  static constexpr int kHistBytes = kWords * NT * 4;
  static constexpr int kRingBytes = RING * RW;
  static constexpr int kWarpBytes = kHistBytes + kRingBytes;
  static constexpr int R2 = (K * K + 1) / 2;        // median rank, 1-based
  static constexpr int E = (G * FW + NT - 1) / NT;  // prefetch bytes per thread
  // byte-lane flags of chunk i that belong to column x (samples 0..K-1) and
  // to column x+1 (samples 1..K)
  __host__ __device__ static constexpr uint32_t mask_lo(int i) {
    uint32_t m = 0;
    for (int b = 0; b < 4; b++)
      if (4 * i + b < K) m |= 0x01u << (8 * b);
    return m;
  }
  __host__ __device__ static constexpr uint32_t mask_hi(int i) {
    uint32_t m = 0;
    for (int b = 0; b < 4; b++)
      if (4 * i + b >= 1 && 4 * i + b <= K) m |= 0x01u << (8 * b);
    return m;
  }
  __host__ __device__ static constexpr uint32_t inc(int j) {
    return j == 0 ? 0x1u : (j == K ? 0x10000u : 0x10001u);
  }
};

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

// One warp per work item (64 output columns x R rows of one channel); the
// warps of a CTA share nothing, so there is no CTA barrier anywhere.
template <int K, int G, int WPC>
__global__ void __launch_bounds__(32 * WPC) hist8_kernel(Job job, int R, int n_strips, int n_segs) {
  using C = HistCfg<K, G>;
  constexpr int NT = C::NT;
  extern __shared__ __align__(16) uint32_t smem[];
  const int warp = threadIdx.x >> 5;
  const int tid = threadIdx.x & 31;
  uint32_t* wbase = smem + warp * (C::kWarpBytes / 4);
  uint8_t* ring = reinterpret_cast<uint8_t*>(wbase + C::kWords * NT);
  constexpr uint32_t kBinStride = 4u * NT;
  const uint32_t hb = smem_u32(wbase + C::kPad * NT + tid);  // bin 0 of this thread
  const int W = job.width, SH = job.src_h, CH = job.channels;
  const int n_items = n_strips * CH * n_segs;

  for (int item = blockIdx.x * WPC + warp; item < n_items; item += gridDim.x * WPC) {
    const int chan = item % CH;
    const int strip = (item / CH) % n_strips;
    const int seg = item / (CH * n_strips);
    const int X0 = strip * 2 * NT;
    const int Y0 = seg * R;
    const int rows = min(R, job.out_h - Y0);
    const uint8_t* src = static_cast<const uint8_t*>(job.src) + chan;
    uint8_t* dst = static_cast<uint8_t*>(job.dst) + chan;
    const int sy_base = job.out_y0 + Y0 - C::H;  // source row of ring row q = 0
    const int q_end = K + rows - 1;              // ring rows of this item: [0, q_end)

    auto fetch = [&](int q0, uint8_t (&v)[C::E]) {
#pragma unroll
      for (int e = 0; e < C::E; e++) {
        const int idx = tid + e * NT;
        const int g = idx / C::FW, c = idx - (idx / C::FW) * C::FW;
        if (idx < G * C::FW && q0 + g < q_end) {
          const int sy = clampi(sy_base + q0 + g, 0, SH - 1);
          const int sx = clampi(X0 - C::H + c, 0, W - 1);
          v[e] = __ldg(src + (int64_t)sy * job.src_pitch + (int64_t)sx * CH);
        }
      }
    };
    auto stash = [&](int q0, const uint8_t (&v)[C::E]) {
#pragma unroll
      for (int e = 0; e < C::E; e++) {
        const int idx = tid + e * NT;
        const int g = idx / C::FW, c = idx - (idx / C::FW) * C::FW;
        if (idx < G * C::FW && q0 + g < q_end) ring[((q0 + g) % C::RING) * C::RW + c] = v[e];
      }
    };

    __syncwarp();  // previous item of this warp done with the ring
    for (int q = 0; q < K + G; q += G) {
      uint8_t v[C::E];
      fetch(q, v);
      stash(q, v);
    }
    for (int b = -C::kPad; b < 256 + C::kPad; b++) st_hist(hb + b * kBinStride, 0u);
    __syncwarp();

    // Samples 0..K of ring row q for this thread (footprint columns 2*tid ..
    // 2*tid + K) as 4-byte chunks.
    auto row_chunks = [&](int q, uint32_t (&ch)[C::NC]) {
      const uint8_t* rp = ring + (q % C::RING) * C::RW;
      const uint32_t* wp = reinterpret_cast<const uint32_t*>(rp) + (tid >> 1);
      const int sh = 16 * (tid & 1);
      uint32_t w[C::NWD];
#pragma unroll
      for (int i = 0; i < C::NWD; i++) w[i] = wp[i];
#pragma unroll
      for (int i = 0; i < C::NC; i++) ch[i] = __funnelshift_r(w[i], w[i + 1], sh);
    };
    auto addr_of = [&](const uint32_t (&ch)[C::NC], int j) -> uint32_t {
      return hb + __byte_perm(ch[j >> 2], 0u, 0x4440 | (j & 3)) * kBinStride;
    };

    // ---- build the first window: rows q = 0 .. K-1 ------------------------
    for (int q = 0; q < K; q++) {
      uint32_t ch[C::NC];
      row_chunks(q, ch);
#pragma unroll
      for (int j = 0; j <= K; j++) red_add(addr_of(ch, j), C::inc(j));
    }

    // Per column c in {0, 1}: m[c] = median bin, bl[c] = #samples < m[c].
    // One round evaluates 8 bins in each column's direction; converged lanes
    // recompute the same state (idempotent), so the warp loops until all agree.
    int m[2] = {128, 128}, bl[2];
    {
      // first window: below(128) from scratch
#pragma unroll
      for (int c = 0; c < 2; c++) {
        int acc = 0;
        for (int b = 0; b < 128; b++) acc += (int)((ld_hist(hb + b * kBinStride) >> (16 * c)) & 0xFFFFu);
        bl[c] = acc;
      }
    }
    auto walk = [&]() {
      constexpr int S = 8;
      for (;;) {
        bool fin[2];
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const bool down = bl[c] >= C::R2;
          const int s1 = down ? -1 : 1;
          const uint32_t a0 = hb + (uint32_t)(down ? m[c] - 1 : m[c]) * kBinStride;
          const uint32_t da = down ? (uint32_t)(-(int)kBinStride) : kBinStride;
          int t[S];
          int acc = bl[c];
          int nlt = 0, best = down ? -1 : bl[c];
#pragma unroll
          for (int i = 0; i < S; i++) {
            const int h = (int)((ld_hist(a0 + i * da) >> (16 * c)) & 0xFFFFu);
            acc += s1 * h;
            t[i] = acc;
          }
#pragma unroll
          for (int i = 0; i < S; i++) {
            const bool lt = t[i] < C::R2;
            nlt += lt;
            best = lt ? max(best, t[i]) : best;  // largest prefix still below rank
          }
          // up: bins m .. m+nlt-1 lie wholly below rank R2 -> median at m + nlt
          // down: bins m-1 .. m-(S-nlt) lie wholly at/above it -> median at
          //       m - (S - nlt) - 1 ... i.e. the first bin whose prefix drops below
          const int nge = S - nlt;
          if (down) {
            fin[c] = nlt > 0;
            m[c] -= fin[c] ? nge + 1 : S;
            bl[c] = fin[c] ? best : t[S - 1];
          } else {
            fin[c] = nlt < S;
            m[c] += nlt;
            bl[c] = fin[c] ? best : t[S - 1];
          }
        }
        if (__all_sync(0xffffffffu, fin[0] && fin[1])) break;
      }
    };
    const int x = X0 + 2 * tid;
    auto store = [&](int yrel) {
      uint8_t* d = dst + (int64_t)(Y0 + yrel) * job.dst_pitch + (int64_t)x * CH;
      if (x < W) d[0] = (uint8_t)m[0];
      if (x + 1 < W) d[CH] = (uint8_t)m[1];
    };
    walk();
    store(0);

    // ---- sweep down: groups of G output rows --------------------------------
    for (int t0 = 1; t0 < rows; t0 += G) {
      uint8_t nxt[C::E];
      const int qn = K + t0 - 1 + G;  // first ring row of the next group
      if (qn < q_end) fetch(qn, nxt);
      const int t1 = min(t0 + G, rows);
      for (int t = t0; t < t1; t++) {
        uint32_t co[C::NC], ci[C::NC];
        row_chunks(t - 1, co);
        row_chunks(t - 1 + K, ci);
#pragma unroll
        for (int j = 0; j <= K; j++) {
          red_add(addr_of(co, j), 0u - C::inc(j));
          red_add(addr_of(ci, j), C::inc(j));
        }
        // below[c] += #entering < m[c] - #leaving < m[c] (before m moves)
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const uint32_t mb = (uint32_t)m[c] * 0x01010101u;
          uint32_t ai = 0, ao = 0;
#pragma unroll
          for (int i = 0; i < C::NC; i++) {
            const uint32_t mk = c ? C::mask_hi(i) : C::mask_lo(i);
            ai += __vsetltu4(ci[i], mb) & mk;
            ao += __vsetltu4(co[i], mb) & mk;
          }
          bl[c] += (int)__dp4a(ai, 0x01010101u, 0u) - (int)__dp4a(ao, 0x01010101u, 0u);
        }
        walk();
        store(t);
      }
      if (qn < q_end) stash(qn, nxt);
      __syncwarp();
    }
  }
}

// Warps per CTA: 1 (CTAs are independent anyway; the hardware packs as many
// as shared memory allows onto each SM).
template <int K>
constexpr int hist_g() { return K <= 31 ? 8 : 4; }

template <int K>
int launch_hist8_k(const Job& job, cudaStream_t stream) {
  constexpr int G = hist_g<K>(), WPC = 1;
  using C = HistCfg<K, G>;
  constexpr int kSmem = C::kWarpBytes * WPC;
  static_assert(kSmem <= 227 * 1024, "histogram kernel does not fit in shared memory");
  auto fn = hist8_kernel<K, G, WPC>;
  static int occ = -1;
  static int sms = 0;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return (int)e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 32 * WPC, kSmem);
    occ = o > 0 ? o : 1;
  }
  const int n_strips = (job.width + 63) / 64;
  const long slots = (long)sms * occ * WPC;  // concurrent warps
  // Row segment length: long enough to amortise the k x k build (about k rows
  // of work), short enough that the last wave is small -- the candidate with
  // the smallest estimated makespan.
  int best_R = job.out_h;
  long best_cost = 0x7fffffffffffL;
  for (int R = 16; R <= 16384; R *= 2) {
    const long segs = (job.out_h + R - 1) / R;
    const long items = segs * n_strips * job.channels;
    const long waves = (items + slots - 1) / slots;
    const long cost = waves * (long)(min(R, job.out_h) + K + 8);
    if (cost < best_cost) {
      best_cost = cost;
      best_R = R;
    }
    if (R >= job.out_h) break;
  }
  const int R = best_R;
  const int n_segs = (job.out_h + R - 1) / R;
  const long items = (long)n_segs * n_strips * job.channels;
  const long ctas = (items + WPC - 1) / WPC;
  const int grid = (int)(ctas < slots / WPC ? ctas : slots / WPC);
  fn<<<grid, 32 * WPC, kSmem, stream>>>(job, R, n_strips, n_segs);
  return (int)cudaGetLastError();
}

template <int... Ks>
struct Hist8Table {
  static int launch(int k, const Job& job, cudaStream_t s) {
    int rc = (int)cudaErrorInvalidValue;
    ((k == Ks ? (rc = launch_hist8_k<Ks>(job, s), 0) : 0), ...);
    return rc;
  }
};

using Hist8All = Hist8Table<3, 5, 7, 9, 11, 13, 15, 17, 19, 21, 23, 25, 27, 29, 31, 33, 35, 37,
                            39, 41, 43, 45, 47, 49, 51, 53, 55, 57, 59, 61, 63, 65, 67, 69, 71,
                            73, 75>;

}  // namespace

bool hist8_supports(int k) { return k >= 3 && k <= 75 && (k & 1); }

int launch_hist8(const Job& job, int k, cudaStream_t s) {
  if (!hist8_supports(k)) return (int)cudaErrorInvalidValue;
  return Hist8All::launch(k, job, s);
}

}  // namespace tmb
