// tm_oblivious.cuh -- data-oblivious hierarchical-tiling median kernel.
//
// Variant (1) of the north star: one register-resident selection program per
// thread (section 4.3; reference stand-in oblivious.py:329-394).
//
// CTA layout (all sizes compile-time):
//   * each thread owns BY x BX-grid position (bx, by) and runs the generated
//     program for one TW x TH root tile *per lane*: two tiles at once for 8/16
//     bit data (u16x2 lane words, lane 1 = the tile OH rows below), one for 32;
//   * stage 1 loads the CTA footprint from global memory into shared memory,
//     clamping coordinates to the image (replicate borders, reference
//     reference.py:37-38 / oblivious.py:362-366), converting to lane words;
//   * stage 2 sorts every footprint column at core height once per tile row,
//     cooperatively (the paper's "collaborative column sort", PAPER.md
//     section 4.3 step 2; reference oblivious.py:368-376), so horizontally
//     adjacent tiles share them;
//   * stage 3 runs the generated straight-line min/max program (program.py /
//     codegen.py) reading raw pixels and sorted columns from shared memory;
//   * stage 4 writes the TW x TH medians of each lane, masking the image edge.
//
// Shared-memory layout: every tile row `by` gets its own block of footprint
// rows and of sorted columns, each block padded to a stride == 1 (mod 32)
// words.  Threads map to tiles as by = tid % BY, bx = tid / BY, so with
// BY == TW the 32 lanes of a warp hit 32 distinct banks on every program load.
#pragma once
#include "tm_common.cuh"

namespace tmb {

template <int N>
struct ColSort;  // generated: static void run(uint32_t (&v)[N]) with Ops policy

template <typename T, int KW, int KH, int TW, int TH>
struct OblGeom {
  static constexpr int HW = KW / 2, HH = KH / 2;
  static constexpr int CH = KH - TH + 1;  // core height = sorted column length
  static constexpr int FWT = KW + TW - 1; // footprint width of one tile
  static constexpr int FHT = KH + TH - 1; // footprint height of one tile
};

__host__ __device__ constexpr int stride_1mod32(int words) {
  return words + ((33 - (words & 31)) & 31);
}

template <typename T, int KW, int KH, int TW, int TH, int BX, int BY>
struct OblLayout {
  using G = OblGeom<T, KW, KH, TW, TH>;
  static constexpr int kLanes = Lanes<T>::kLanes;
  static constexpr int kThreads = BX * BY;
  static constexpr int OW = BX * TW;             // output columns per CTA
  static constexpr int OH = BY * TH;             // output rows per lane per CTA
  static constexpr int FW = OW + KW - 1;         // footprint columns per CTA
  static constexpr int RB = stride_1mod32(G::FHT * FW);   // raw block stride (per tile row)
  static constexpr int SB = stride_1mod32(G::CH * FW);    // sorted-column block stride
  static constexpr int kSmemWords = BY * RB + BY * SB;
  static constexpr int kSmemBytes = kSmemWords * 4;
};

// Program I/O: the generated code calls pix(x, y) / col(x, i) with compile-time
// offsets relative to the tile anchor, mn/mx for the lane min/max and out().
template <typename T, int KW, int KH, int TW, int TH, int BX, int BY>
struct OblIO {
  using Lay = OblLayout<T, KW, KH, TW, TH, BX, BY>;
  using G = OblGeom<T, KW, KH, TW, TH>;
  const uint32_t* raw;   // at (tile-row block, footprint row 0, tile column 0)
  const uint32_t* scol;  // at (tile-row block, i = 0, tile column 0)
  uint32_t res[TH][TW];
  // x, y relative to the tile anchor; the tile footprint starts at (-HW, -HH)
  __device__ __forceinline__ uint32_t pix(int x, int y) const {
    return raw[(y + G::HH) * Lay::FW + (x + G::HW)];
  }
  __device__ __forceinline__ uint32_t col(int x, int i) const {
    return scol[i * Lay::FW + (x + G::HW)];
  }
  __device__ __forceinline__ static uint32_t mn(uint32_t a, uint32_t b) { return Lanes<T>::mn(a, b); }
  __device__ __forceinline__ static uint32_t mx(uint32_t a, uint32_t b) { return Lanes<T>::mx(a, b); }
  __device__ __forceinline__ void out(int x, int y, uint32_t v) { res[y][x] = v; }
};

template <typename T, int KW, int KH, int TW, int TH, int BX, int BY, class Prog, class CSort>
__global__ void __launch_bounds__(BX * BY)
obl_kernel(Job job) {
  using Lay = OblLayout<T, KW, KH, TW, TH, BX, BY>;
  using G = OblGeom<T, KW, KH, TW, TH>;
  using L = Lanes<T>;
  constexpr int NT = Lay::kThreads;
  extern __shared__ uint32_t smem[];
  uint32_t* raw = smem;
  uint32_t* scol = smem + BY * Lay::RB;

  const int tid = threadIdx.x;
  const int X0 = blockIdx.x * Lay::OW;
  const int Y0 = blockIdx.y * Lay::OH * Lay::kLanes;  // output row (band-relative) of lane 0
  const int W = job.width, SH = job.src_h;
  const int sy0 = job.out_y0 + Y0;                     // source row of lane 0's first output

  // ---- stage 1: footprint -> shared memory (one block per tile row) -------
  constexpr int kRawItems = BY * G::FHT * Lay::FW;
  for (int idx = tid; idx < kRawItems; idx += NT) {
    const int rx = idx % Lay::FW;
    const int t = idx / Lay::FW;
    const int ry = t % G::FHT;
    const int by = t / G::FHT;
    const int gx = clampi(X0 + rx - G::HW, 0, W - 1);
    const int yy = by * TH + ry - G::HH;
    const T a = load_px<T>(job, clampi(sy0 + yy, 0, SH - 1), gx);
    T b = a;
    if (Lay::kLanes == 2) b = load_px<T>(job, clampi(sy0 + Lay::OH + yy, 0, SH - 1), gx);
    raw[by * Lay::RB + ry * Lay::FW + rx] = L::pack(a, b);
  }
  __syncthreads();

  // ---- stage 2: cooperative column sorts at core height ------------------
  constexpr int kColItems = BY * Lay::FW;
  for (int idx = tid; idx < kColItems; idx += NT) {
    const int rx = idx % Lay::FW;
    const int by = idx / Lay::FW;
    uint32_t v[G::CH];
    const uint32_t* src = raw + by * Lay::RB + (TH - 1) * Lay::FW + rx;
#pragma unroll
    for (int i = 0; i < G::CH; i++) v[i] = src[i * Lay::FW];
    CSort::template run<L>(v);
    uint32_t* dst = scol + by * Lay::SB + rx;
#pragma unroll
    for (int i = 0; i < G::CH; i++) dst[i * Lay::FW] = v[i];
  }
  __syncthreads();

  // ---- stage 3: per-thread selection program -----------------------------
  const int by = tid % BY;
  const int bx = tid / BY;
  OblIO<T, KW, KH, TW, TH, BX, BY> io;
  io.raw = raw + by * Lay::RB + bx * TW;
  io.scol = scol + by * Lay::SB + bx * TW;
  Prog::run(io);

  // ---- stage 4: store (masked at the image / band edge) -------------------
#pragma unroll
  for (int l = 0; l < Lay::kLanes; l++) {
#pragma unroll
    for (int y = 0; y < TH; y++) {
      const int oy = Y0 + l * Lay::OH + by * TH + y;
      if (oy >= job.out_h) continue;
#pragma unroll
      for (int x = 0; x < TW; x++) {
        const int ox = X0 + bx * TW + x;
        if (ox < W) store_px<T>(job, oy, ox, (T)L::lane(io.res[y][x], l));
      }
    }
  }
}

}  // namespace tmb
