// tm_hist.cu -- data-aware O(k) median for 8-bit images: per-column sliding
// histograms swept down the image (variant (2) for uint8).
//
// Reference role: the data-aware engine (aware.py:437-492, section 5)
// reuses sorted runs between neighbouring output pixels so the work per pixel
// grows O(k) instead of O(k^2).  For 8-bit data the cheapest shareable
// structure on a GPU is the window histogram itself: moving the k x k window
// one row down removes k samples and adds k samples, and the median (rank
// r = (k^2+1)/2, geometry.py:55-58) is found by walking from the previous
// median, which rarely moves far.  Results are exact by construction: the
// histogram is the window's multiset.
//
// Layout (one CTA = NT adjacent output columns x one segment of R output rows
// of one channel; a grid-stride loop over (row segment, column strip,
// channel) work items keeps every SM busy to the last item):
//   * hist: per thread 256 bins x one 32-bit word, word (bin, thread) at
//     bin * NT + tid -- a warp's accesses hit 32 distinct banks whatever the
//     bins.  Each word holds HS sub-histograms (u8 x 4 for k <= 31, u16 x 2
//     above): window column j counts into sub-histogram j % HS, so HS
//     read-modify-write chains per thread run concurrently (the chains are
//     independent because they touch different bytes);
//   * ring: the last k + G + 1 source rows of the strip's footprint
//     (NT + k - 1 samples each, clamped = replicate borders), refilled G rows
//     at a time.
// Per output row a thread removes the leaving row's k samples and adds the
// entering row's k samples (one LDS/STS pair per sample, k/HS dependent
// round trips), keeps `below` = #samples < m incrementally and walks m to the
// bin holding rank r.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tm_common.cuh"
#include "tm_kernels.h"

namespace tmb {
namespace {

// Update modes (template MODE):
//   0: LDS/STS read-modify-write, 4 (k <= 31, u8 counts) or 2 (u16 counts)
//      sub-histograms per bin word, one round trip per HS window columns;
//   1: RED.ADD (shared atomic without return) on one u32 count per bin --
//      no round trip, no aliasing hazard;
//   2: RED.ADD on u16 counts, bins (2w, 2w+1) in word w -- half the shared
//      memory of mode 1 (twice the threads per SM).
template <int K, int NT, int G, int MODE>
struct HistCfg {
  static constexpr int H = K / 2;
  static constexpr bool kWide = K > 31;             // mode 0: u16 counts
  static constexpr int HS = MODE == 0 ? (kWide ? 2 : 4) : 1;
  static constexpr int CS = kWide ? 2 : 1;          // mode 0: bytes per count
  static constexpr int RING = K + 2 * G + 1;        // next group stored while this one runs
  static constexpr int FW = NT + K - 1;             // footprint columns
  static constexpr int RW = ((FW + 3) / 4) * 4 + 8; // ring row bytes (+ slack words)
  static constexpr int NWD = (K + 3) / 4 + 1;       // aligned words covering k bytes
  static constexpr int kPad = 4;                    // zero bins below 0 / above 255
  static constexpr int kWords = MODE == 2 ? (256 + 2 * kPad) / 2 : 256 + 2 * kPad;
  static constexpr int kHistBytes = kWords * NT * 4;
  static constexpr int kRingBytes = RING * RW;
  static constexpr int kSmem = kHistBytes + kRingBytes;
  static constexpr int R2 = (K * K + 1) / 2;        // median rank, 1-based
  static constexpr int E = (G * FW + NT - 1) / NT;  // prefetch bytes per thread
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Histogram memory operations.  VOL selects ld/st.volatile (never reordered
// against each other by ptxas) or plain accesses.
template <int CS, bool VOL>
struct SmemOps;

#define TMB_SMEM_OPS(CS_, SUF, VOLB, Q)                                            \
  template <>                                                                     \
  struct SmemOps<CS_, VOLB> {                                                     \
    __device__ __forceinline__ static uint32_t ld(uint32_t a) {                   \
      uint32_t v;                                                                 \
      asm volatile("ld" Q ".shared." SUF " %0, [%1];" : "=r"(v) : "r"(a) : "memory"); \
      return v;                                                                   \
    }                                                                             \
    __device__ __forceinline__ static void st(uint32_t a, uint32_t v) {           \
      asm volatile("st" Q ".shared." SUF " [%0], %1;" ::"r"(a), "r"(v) : "memory"); \
    }                                                                             \
  };
TMB_SMEM_OPS(1, "u8", true, ".volatile")
TMB_SMEM_OPS(1, "u8", false, "")
TMB_SMEM_OPS(2, "u16", true, ".volatile")
TMB_SMEM_OPS(2, "u16", false, "")
TMB_SMEM_OPS(4, "u32", true, ".volatile")
TMB_SMEM_OPS(4, "u32", false, "")
#undef TMB_SMEM_OPS

__device__ __forceinline__ void red_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

template <int K, int NT, int G, int MODE, int ORD>
__global__ void __launch_bounds__(NT) hist8_kernel(Job job, int R, int n_strips, int n_segs) {
  using C = HistCfg<K, NT, G, MODE>;
  // ORD (experiments on update/walk ordering): 0 volatile everything,
  // 1 plain, 2 plain + __syncwarp before the walk, 3 plain + membar.cta before
  // the walk, 4 volatile updates + plain walk loads.
  constexpr bool kVolUpd = ORD == 0 || ORD == 4;
  constexpr bool kVolWalk = ORD == 0;
  using Ops = SmemOps<C::CS, kVolUpd>;
  using W32 = SmemOps<4, kVolWalk>;
  using Z32 = SmemOps<4, kVolUpd>;
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* hist = smem;  // [kWords][NT]
  uint8_t* ring = reinterpret_cast<uint8_t*>(smem + C::kWords * NT);
  const int tid = threadIdx.x;
  constexpr uint32_t kBinStride = 4u * NT;
  // word of bin b (b in [-kPad, 256 + kPad)) of this thread
  const uint32_t* hw = hist + (MODE == 2 ? C::kPad / 2 : C::kPad) * NT + tid;
  const uint32_t hb = smem_u32(hw);
  const int W = job.width, SH = job.src_h, CH = job.channels;
  const int n_items = n_strips * CH * n_segs;

  // All histogram traffic (updates, walk loads, zeroing) is explicit volatile
  // PTX so neither the front end nor ptxas may reorder accesses that alias
  // through data-dependent bin addresses.
  auto count = [&](int b) -> int {
    if constexpr (MODE == 0) {
      const uint32_t w = W32::ld(hb + b * kBinStride);
      if constexpr (C::kWide) return (int)((w & 0xFFFFu) + (w >> 16));
      else return (int)__dp4a(w, 0x01010101u, 0u);
    } else if constexpr (MODE == 1) {
      return (int)W32::ld(hb + b * kBinStride);
    } else {
      const uint32_t w = W32::ld(hb + (b >> 1) * kBinStride);
      return (int)((w >> ((b & 1) << 4)) & 0xFFFFu);
    }
  };

  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int chan = item % CH;
    const int strip = (item / CH) % n_strips;
    const int seg = item / (CH * n_strips);
    const int X0 = strip * NT;
    const int Y0 = seg * R;
    const int rows = min(R, job.out_h - Y0);
    const uint8_t* src = static_cast<const uint8_t*>(job.src) + chan;
    uint8_t* dst = static_cast<uint8_t*>(job.dst) + chan;
    const int sy_base = job.out_y0 + Y0 - C::H;  // source row of ring row q = 0
    // ring rows that exist for this item: q < K + rows - 1
    const int q_end = K + rows - 1;

    // Global loads of ring rows [q0, q0 + G) into registers / into the ring.
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

    __syncthreads();  // previous item done with the ring
    {
      // prologue: the first window (rows 0 .. K-1) and the first group
      for (int q = 0; q < K + G; q += G) {
        uint8_t v[C::E];
        fetch(q, v);
        stash(q, v);
      }
    }
    for (int b = -C::kPad; b < 256 + C::kPad; b += (MODE == 2 ? 2 : 1))
      Z32::st(hb + (MODE == 2 ? b >> 1 : b) * kBinStride, 0u);
    __syncthreads();

    // Read k consecutive samples (footprint columns tid .. tid + K - 1) of
    // ring row q as aligned 4-byte chunks.
    auto row_chunks = [&](int q, uint32_t (&ch)[(K + 3) / 4]) {
      const uint8_t* rp = ring + (q % C::RING) * C::RW;
      const uint32_t* wp = reinterpret_cast<const uint32_t*>(rp) + (tid >> 2);
      const int sh = 8 * (tid & 3);
      uint32_t w[C::NWD];
#pragma unroll
      for (int i = 0; i < C::NWD; i++) w[i] = wp[i];
#pragma unroll
      for (int i = 0; i < (K + 3) / 4; i++) ch[i] = __funnelshift_r(w[i], w[i + 1], sh);
    };
    auto byte_of = [](const uint32_t (&ch)[(K + 3) / 4], int j) -> uint32_t {
      return __byte_perm(ch[j >> 2], 0u, 0x4440 | (j & 3));
    };
    // address / increment of bin v for the RED modes
    auto red_addr = [&](uint32_t v) -> uint32_t {
      if constexpr (MODE == 2) return hb + (v >> 1) * kBinStride;
      else return hb + v * kBinStride;
    };
    auto red_one = [](uint32_t v) -> uint32_t {
      if constexpr (MODE == 2) return 1u << ((v & 1u) << 4);
      else return 1u;
    };

    // ---- build the first window: rows q = 0 .. K-1 ------------------------
    for (int q = 0; q < K; q++) {
      uint32_t ch[(K + 3) / 4];
      row_chunks(q, ch);
      if constexpr (MODE == 0) {
#pragma unroll
        for (int j0 = 0; j0 < K; j0 += C::HS) {
          uint32_t a[C::HS], c[C::HS];
#pragma unroll
          for (int s = 0; s < C::HS; s++)
            if (j0 + s < K) a[s] = hb + byte_of(ch, j0 + s) * kBinStride + s * C::CS;
#pragma unroll
          for (int s = 0; s < C::HS; s++)
            if (j0 + s < K) c[s] = Ops::ld(a[s]);
#pragma unroll
          for (int s = 0; s < C::HS; s++)
            if (j0 + s < K) Ops::st(a[s], c[s] + 1);
        }
      } else {
#pragma unroll
        for (int j = 0; j < K; j++) {
          const uint32_t v = byte_of(ch, j);
          red_add(red_addr(v), red_one(v));
        }
      }
    }
    int m = 0;
    int below = 0;
    // Move m to the bin holding rank R2 (below = #samples < m), 4 bins per
    // round trip.
    auto walk = [&]() {
      // Warp-convergent: every lane evaluates 4 bins per round in its own
      // direction; a lane whose bin already holds rank R2 recomputes the same
      // state (the step is idempotent), so the warp loops until all agree.
      for (;;) {
        const bool down = below >= C::R2;
        const int s1 = down ? -1 : 1;
        const int b0 = down ? m - 1 : m;
        const int h0 = count(b0), h1 = count(b0 + s1), h2 = count(b0 + 2 * s1),
                  h3 = count(b0 + 3 * s1);
        const int d0 = s1 * h0, d1 = s1 * h1, d2 = s1 * h2, d3 = s1 * h3;
        const int t0 = below + d0, t1 = t0 + d1, t2 = t1 + d2, t3 = t2 + d3;
        int n;
        if (down) n = (t0 >= C::R2) + (t1 >= C::R2) + (t2 >= C::R2) + (t3 >= C::R2);
        else n = (t0 < C::R2) + (t1 < C::R2) + (t2 < C::R2) + (t3 < C::R2);
        // up: median in bin m + n (n < 4), below = t_{n-1} (or below);
        // down: median in bin m - 1 - n (n < 4), below = t_n.
        const int tn1 = n == 0 ? below : n == 1 ? t0 : n == 2 ? t1 : n == 3 ? t2 : t3;
        const int tn = n == 0 ? t0 : n == 1 ? t1 : n == 2 ? t2 : t3;
        const bool fin = n < 4;
        if (down) {
          m -= fin ? n + 1 : 4;
          below = tn;
        } else {
          m += n;
          below = fin ? tn1 : t3;
        }
        if (__all_sync(0xffffffffu, fin)) break;
      }
    };
    walk();
    const int x = X0 + tid;
    const bool col_ok = x < W;
    if (col_ok) dst[(int64_t)Y0 * job.dst_pitch + (int64_t)x * CH] = (uint8_t)m;

    // ---- sweep down: groups of G output rows --------------------------------
    for (int t0 = 1; t0 < rows; t0 += G) {
      uint8_t nxt[C::E];
      const int qn = K + t0 - 1 + G;  // first ring row of the next group
      if (qn < q_end) fetch(qn, nxt);
      const int t1 = min(t0 + G, rows);
      for (int t = t0; t < t1; t++) {
        uint32_t co[(K + 3) / 4], ci[(K + 3) / 4];
        row_chunks(t - 1, co);
        row_chunks(t - 1 + K, ci);
        if constexpr (MODE == 0) {
#pragma unroll
          for (int j0 = 0; j0 < K; j0 += C::HS) {
            uint32_t ao[C::HS], ai[C::HS], same[C::HS], c_o[C::HS], c_i[C::HS];
#pragma unroll
            for (int s = 0; s < C::HS; s++) {
              if (j0 + s < K) {
                const uint32_t vo = byte_of(co, j0 + s), vi = byte_of(ci, j0 + s);
                below += (int)((uint32_t)((int)vi - m) >> 31) - (int)((uint32_t)((int)vo - m) >> 31);
                ao[s] = hb + vo * kBinStride + s * C::CS;
                ai[s] = hb + vi * kBinStride + s * C::CS;
                same[s] = vo == vi;
              }
            }
#pragma unroll
            for (int s = 0; s < C::HS; s++)
              if (j0 + s < K) {
                c_o[s] = Ops::ld(ao[s]);
                c_i[s] = Ops::ld(ai[s]);
              }
#pragma unroll
            for (int s = 0; s < C::HS; s++)
              if (j0 + s < K) Ops::st(ao[s], c_o[s] - 1);
#pragma unroll
            for (int s = 0; s < C::HS; s++)
              if (j0 + s < K) Ops::st(ai[s], c_i[s] + 1 - same[s]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < K; j++) {
            const uint32_t vo = byte_of(co, j), vi = byte_of(ci, j);
            below += (int)((uint32_t)((int)vi - m) >> 31) - (int)((uint32_t)((int)vo - m) >> 31);
            red_add(red_addr(vo), 0u - red_one(vo));
            red_add(red_addr(vi), red_one(vi));
          }
        }
        if constexpr (ORD == 2) __syncwarp();
        if constexpr (ORD == 3) __threadfence_block();
        walk();
        if (col_ok) dst[(int64_t)(Y0 + t) * job.dst_pitch + (int64_t)x * CH] = (uint8_t)m;
      }
      if (qn < q_end) stash(qn, nxt);
      __syncthreads();
    }
  }
}

template <int K, int NT, int MODE, int ORD>
int launch_hist8_cfg(const Job& job, cudaStream_t stream) {
  constexpr int G = 8;
  using C = HistCfg<K, NT, G, MODE>;
  auto fn = hist8_kernel<K, NT, G, MODE, ORD>;
  static int occ = -1;
  static int sms = 0;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return (int)e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, NT, C::kSmem);
    occ = o > 0 ? o : 1;
  }
  const int n_strips = (job.width + NT - 1) / NT;
  const int slots = sms * occ;
  // Row segment length: long enough to amortise the k x k build (~k rows of
  // work), short enough that the last wave is small.  Pick the candidate with
  // the smallest estimated makespan.
  int best_R = job.out_h;
  long best_cost = 0x7fffffffffffL;
  for (int R = 32; R <= 8192; R *= 2) {
    const int segs = (job.out_h + R - 1) / R;
    const long items = (long)segs * n_strips * job.channels;
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
  const int grid = (int)(items < slots ? items : slots);
  fn<<<grid, NT, C::kSmem, stream>>>(job, R, n_strips, n_segs);
  return (int)cudaGetLastError();
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <int K, int MODE, int NT>
int launch_hist8_mode(const Job& job, cudaStream_t stream) {
#ifdef TMB_HIST_EXPERIMENT
  if (K == 9 || K == 17 || K == 33) {
    static const int ord = env_int("TMB_HIST_ORD", 0);
    switch (ord) {
      case 1: return launch_hist8_cfg<K, NT, MODE, 1>(job, stream);
      case 2: return launch_hist8_cfg<K, NT, MODE, 2>(job, stream);
      case 3: return launch_hist8_cfg<K, NT, MODE, 3>(job, stream);
      case 4: return launch_hist8_cfg<K, NT, MODE, 4>(job, stream);
      default: break;
    }
  }
#endif
  return launch_hist8_cfg<K, NT, MODE, 0>(job, stream);
}

template <int K>
int launch_hist8_k(const Job& job, cudaStream_t stream) {
  static const int mode = env_int("TMB_HIST_MODE", 2);
  switch (mode) {
    case 0: return launch_hist8_mode<K, 0, 128>(job, stream);
    case 2: return launch_hist8_mode<K, 2, 256>(job, stream);
    default: return launch_hist8_mode<K, 1, 128>(job, stream);
  }
}

template <int... Ks>
struct Hist8Table {
  static int launch(int k, const Job& job, cudaStream_t s) {
    int rc = -1;
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
