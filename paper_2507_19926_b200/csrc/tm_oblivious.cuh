// tm_oblivious.cuh -- data-oblivious hierarchical-tiling median kernel.
//
// Variant (1) of the north star: one register-resident selection program per
// thread (section 4.3; reference stand-in oblivious.py:329-394).
//
// CTA layout (all sizes compile-time):
//   * each thread owns grid position (bx, by) and runs the generated program
//     for one TW x TH root tile *per lane*: two tiles at once for 8/16-bit
//     data (u16x2 lane words, lane 1 = the tile OH rows below), one for 32;
//   * stage 1 loads the CTA footprint from global memory into shared memory,
//     clamping coordinates to the image (replicate borders, reference
//     reference.py:37-38 / oblivious.py:362-366), converting to lane words;
//   * stage 2 sorts every footprint column at core height once per tile row,
//     cooperatively (the paper's "collaborative column sort", PAPER.md
//     section 4.3 step 2; reference oblivious.py:368-376), so horizontally
//     adjacent tiles share them;
//   * stage 3 runs the generated straight-line min/max program (program.py /
//     codegen.py).  It reads raw pixels and sorted columns from shared memory
//     at first use; when the program's live state exceeds its register
//     budget the generator spills computed values to a per-thread shared
//     memory area (slot-major, thread-fastest: bank-conflict free) and
//     reloads them before use -- explicit, Belady-ordered placement instead
//     of ptxas local-memory spills;
//   * each leaf median goes to a shared-memory output tile the moment it is
//     computed; stage 4 writes the tile to global memory coalesced.
//
// Bank conflicts: threads map to tiles as by = tid % BY, bx = tid / BY.  The
// sorted columns of tile row `by` sit in their own block whose stride is
// == 1 (mod 32) words, so with BY == TW a warp's 32 column loads hit 32
// distinct banks; raw rows use a stride == 1 (mod 16).
#pragma once
#include "tm_common.cuh"

namespace tmb {

template <typename T, int KW, int KH, int TW, int TH>
struct OblGeom {
  static constexpr int HW = KW / 2, HH = KH / 2;
  static constexpr int CH = KH - TH + 1;  // core height = sorted column length
};

__host__ __device__ constexpr int stride_1mod32(int words) {
  return words + ((33 - (words & 31)) & 31);
}

template <typename T, int KW, int KH, int TW, int TH, int BX, int BY, int S, int PAIR = 0>
struct OblLayout {
  using G = OblGeom<T, KW, KH, TW, TH>;
  static constexpr int kLanes = Lanes<T>::kLanes;
  static constexpr int kThreads = BX * BY * (PAIR ? 2 : 1);
  static constexpr int OW = BX * TW;             // output columns per CTA
  static constexpr int OH = BY * TH;             // output rows per lane per CTA
  static constexpr int FW = OW + KW - 1;         // footprint columns per CTA
  static constexpr int RH = OH + KH - 1;         // footprint rows per lane
  static constexpr int P = FW + ((17 - (FW & 15)) & 15);  // raw row stride, == 1 (mod 16)
  static constexpr int SB = stride_1mod32(G::CH * P);    // sorted-column block stride
  static constexpr int kRawWords = RH * P;
  static constexpr int kScolWords = BY * SB;
  static constexpr int kSpillWords = S * kThreads;
  static constexpr int kOutWords = OH * OW;
  static constexpr int kSmemWords = kRawWords + kScolWords + kSpillWords + kOutWords;
  static constexpr int kSmemBytes = kSmemWords * 4;
};

// Program I/O: the generated code calls pix(x, y) / col(x, i) with compile-time
// offsets relative to the tile anchor, mn/mx for the lane min/max, spill /
// reload for its shared-memory slots and out() for each leaf median.
template <typename T, class Lay>
struct OblIO {
  using G = typename Lay::G;
  const uint32_t* raw;        // (tile footprint row 0, tile column 0)
  const uint32_t* scol;       // (tile-row block, i = 0, tile column 0)
  volatile uint32_t* spl;     // this thread's slot 0; slot s at spl[s * kThreads]
  uint32_t* outp;             // (tile row 0, tile column 0) of the output tile
  __device__ __forceinline__ uint32_t pix(int x, int y) const {
    return raw[(y + G::HH) * Lay::P + (x + G::HW)];
  }
  __device__ __forceinline__ uint32_t col(int x, int i) const {
    return scol[i * Lay::P + (x + G::HW)];
  }
  __device__ __forceinline__ void spill(int s, uint32_t v) const { spl[s * Lay::kThreads] = v; }
  __device__ __forceinline__ uint32_t reload(int s) const { return spl[s * Lay::kThreads]; }
  __device__ __forceinline__ static uint32_t mn(uint32_t a, uint32_t b) { return Lanes<T>::mn(a, b); }
  __device__ __forceinline__ static uint32_t mx(uint32_t a, uint32_t b) { return Lanes<T>::mx(a, b); }
  __device__ __forceinline__ void out(int x, int y, uint32_t v) const { outp[y * Lay::OW + x] = v; }
};

// Pair I/O (pairgen.py): thread `role` of a lane pair works on one root tile;
// *_t accessors translate the root-phase halves, *_m mirror the child phase
// (x -> TW-1-x for role 1), xchg swaps a value with the partner lane.
template <typename T, class Lay, class Prog>
struct PairIO {
  using G = typename Lay::G;
  const uint32_t* raw_t;   // root phase rows: footprint row 0 + role * kRowShift
  const uint32_t* col_tb;  // root phase core halves: + role * kCoreHalf columns
  const uint32_t* raw_m;   // child phase: mirrored column origin
  const uint32_t* col_mb;
  uint32_t* out_mb;
  int s;                   // +1 (role 0) or -1 (role 1)
  int role;
  __device__ __forceinline__ uint32_t pix_t(int x, int y) const {
    return raw_t[(y + G::HH) * Lay::P + (x + G::HW)];
  }
  __device__ __forceinline__ uint32_t col_t(int x, int i) const {
    return col_tb[i * Lay::P + (x + G::HW)];
  }
  __device__ __forceinline__ uint32_t pix_m(int x, int y) const {
    return raw_m[(y + G::HH) * Lay::P + s * x];
  }
  __device__ __forceinline__ uint32_t col_m(int x, int i) const {
    return col_mb[i * Lay::P + s * x];
  }
  __device__ __forceinline__ void out_m(int x, int y, uint32_t v) const {
    out_mb[y * Lay::OW + s * x] = v;
  }
  __device__ __forceinline__ static uint32_t xchg(uint32_t v) { return __shfl_xor_sync(0xffffffffu, v, 1); }
  __device__ __forceinline__ uint32_t sel(uint32_t a, uint32_t b) const { return role ? b : a; }
  __device__ __forceinline__ static uint32_t mn(uint32_t a, uint32_t b) { return Lanes<T>::mn(a, b); }
  __device__ __forceinline__ static uint32_t mx(uint32_t a, uint32_t b) { return Lanes<T>::mx(a, b); }
};

template <typename T, int KW, int KH, int TW, int TH, int BX, int BY, class Prog, class CSort>
__global__ void __launch_bounds__(BX * BY * (Prog::kPair ? 2 : 1))
obl_kernel(Job job0) {
  using Lay = OblLayout<T, KW, KH, TW, TH, BX, BY, Prog::kSpillSlots, Prog::kPair>;
  // channels are interleaved into blockIdx.x (c fastest) so the CTAs of all
  // planes of one image region run together and share L2 sectors of the
  // interleaved (H, W, C) buffer -- both for the loads and the byte stores
  Job job = job0;
  const int chan = blockIdx.x % job0.channels;
  const int tile_x = blockIdx.x / job0.channels;
  job.src = static_cast<const T*>(job0.src) + chan;
  job.dst = static_cast<T*>(job0.dst) + chan;
  using G = OblGeom<T, KW, KH, TW, TH>;
  using L = Lanes<T>;
  constexpr int NT = Lay::kThreads;
  extern __shared__ uint32_t smem[];
  uint32_t* raw = smem;
  uint32_t* scol = raw + Lay::kRawWords;
  uint32_t* spill = scol + Lay::kScolWords;
  uint32_t* outt = spill + Lay::kSpillWords;

  const int tid = threadIdx.x;
  const int X0 = tile_x * Lay::OW;
  const int Y0 = blockIdx.y * Lay::OH * Lay::kLanes;  // output row (band-relative) of lane 0
  const int W = job.width, SH = job.src_h;
  const int sy0 = job.out_y0 + Y0 - G::HH;             // source row of footprint row 0, lane 0

  // ---- stage 1: footprint -> shared memory lane words ---------------------
  // Every thread issues all of its global loads before consuming any (the
  // CTA's footprint is loaded with E loads in flight per thread instead of
  // one round trip per element), then packs and stores them.
  {
    constexpr int kItems = Lay::RH * Lay::FW;
    constexpr int E = (kItems + NT - 1) / NT;
    T va[E], vb[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
      const int idx = tid + e * NT;
      const int r = idx / Lay::FW, c = idx - (idx / Lay::FW) * Lay::FW;
      if (idx < kItems) {
        const int gx = clampi(X0 + c - G::HW, 0, W - 1);
        va[e] = load_px<T>(job, clampi(sy0 + r, 0, SH - 1), gx);
        vb[e] = Lay::kLanes == 2 ? load_px<T>(job, clampi(sy0 + Lay::OH + r, 0, SH - 1), gx) : va[e];
      }
    }
#pragma unroll
    for (int e = 0; e < E; e++) {
      const int idx = tid + e * NT;
      const int r = idx / Lay::FW, c = idx - (idx / Lay::FW) * Lay::FW;
      if (idx < kItems) raw[r * Lay::P + c] = L::pack(va[e], vb[e]);
    }
  }
  __syncthreads();

  // ---- stage 2: cooperative column sorts at core height ------------------
  constexpr int kColItems = BY * Lay::FW;
  for (int idx = tid; idx < kColItems; idx += NT) {
    const int by = idx / Lay::FW;
    const int rx = idx - by * Lay::FW;
    uint32_t v[G::CH];
    const uint32_t* src = raw + (by * TH + TH - 1) * Lay::P + rx;
#pragma unroll
    for (int i = 0; i < G::CH; i++) v[i] = src[i * Lay::P];
    CSort::template run<L>(v);
    uint32_t* dst = scol + by * Lay::SB + rx;
#pragma unroll
    for (int i = 0; i < G::CH; i++) dst[i * Lay::P] = v[i];
  }
  __syncthreads();

  // ---- stage 3: per-thread selection program -----------------------------
  if constexpr (Prog::kPair) {
    const int role = tid & 1, pr = tid >> 1;
    const int by = pr % BY;
    const int bx = pr / BY;
    const uint32_t* rt = raw + by * TH * Lay::P + bx * TW;
    const uint32_t* st = scol + by * Lay::SB + bx * TW;
    PairIO<T, Lay, Prog> io;
    io.role = role;
    io.s = 1 - 2 * role;
    io.raw_t = rt + role * Prog::kRowShift * Lay::P;
    io.col_tb = st + role * Prog::kCoreHalf;
    io.raw_m = rt + G::HW + role * (TW - 1);
    io.col_mb = st + G::HW + role * (TW - 1);
    io.out_mb = outt + by * TH * Lay::OW + bx * TW + role * (TW - 1);
    Prog::run(io);
  } else {
    const int by = tid % BY;
    const int bx = tid / BY;
    OblIO<T, Lay> io;
    io.raw = raw + by * TH * Lay::P + bx * TW;
    io.scol = scol + by * Lay::SB + bx * TW;
    io.spl = spill + tid;
    io.outp = outt + by * TH * Lay::OW + bx * TW;
    Prog::run(io);
  }
  __syncthreads();

  // ---- stage 4: coalesced store of the output tile ------------------------
#pragma unroll
  for (int l = 0; l < Lay::kLanes; l++) {
    for (int idx = tid; idx < Lay::OH * Lay::OW; idx += NT) {
      const int y = idx / Lay::OW, x = idx - y * Lay::OW;
      const int oy = Y0 + l * Lay::OH + y, ox = X0 + x;
      if (oy < job.out_h && ox < W) store_px<T>(job, oy, ox, (T)L::lane(outt[idx], l));
    }
  }
}

}  // namespace tmb
