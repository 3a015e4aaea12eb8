// tm_aware.cu -- data-aware multi-pass hierarchical-tiling median (variant 2).
//
// The paper's large-kernel implementation (section 5.3, Fig. 5 compute
// graph: row sort, column sort, core sort, row / column / core extension,
// finalization) with the reference's pass structure (aware.py:176-492):
//
//   pass_init          (aware.py:239-286)  sort_runs (rows, cols) + core merge
//   pass_extend_level  (aware.py:289-373)  fused horizontal + vertical split:
//                                          pack merges, trimmed candidate
//                                          merges, row / column extension
//   pass_finalize      (aware.py:376-413)  per pixel: select the median rank
//                                          from cand + column run + row run +
//                                          corner (binary-search selection in
//                                          four sorted arrays)
//
// Every buffer lives in device memory (stream-ordered cudaMallocAsync); bands
// of root-tile rows bound the footprint exactly like the reference's
// slice_budget banding (aware.py:455-463).  All merges -- the k-way packs
// (binary reduction), the trimmed candidate merges and the run extensions --
// go through ONE batched merge kernel: each thread finds its output range's
// merge-path split by binary search (ties go to A, aware.py:62-85) and then
// merges sequentially.  Tie order never changes values, so every candidate
// window is the reference's window value for value.
#include <algorithm>
#include <cstdio>
#include <mutex>
#include <vector>

#include "tm_common.cuh"
#include "tm_kernels.h"

namespace tmb {
namespace aware {

// ------------------------------------------------------------------------
// geometry helpers (host + device)

struct Win {
  int lo, hi;  // 1-based ranks among the seen values
};

__host__ __device__ inline Win retention(long n_total, long n_seen) {
  const long r = (n_total + 1) / 2, m = n_total - n_seen;
  Win w;
  w.lo = (int)(r - m > 1 ? r - m : 1);
  w.hi = (int)(n_seen < r ? n_seen : r);
  return w;
}

inline int root_tile(int k) {
  int b = 0;
  while ((1 << (b + 1)) <= k) b++;  // floor(log2 k)
  int t = 1 << (b - 1);
  return t < 2 ? 2 : t;
}

// Offset of batched problem m: ((m / D) >> SH1) * S1 + ((m % D) >> SH2) * S2.
// Covers contiguous problems and the "parent = child / 2" patterns of a split.
struct Addr {
  long s1, s2;
  int d, sh1, sh2;
  __host__ __device__ long at(long m) const {
    return ((m / d) >> sh1) * s1 + ((m % d) >> sh2) * s2;
  }
};

inline Addr lin(long stride) { return Addr{stride, 0, 1, 0, 0}; }

// ------------------------------------------------------------------------
// batched merge: out_m[0, cnt) = merge(A_m[0, p), B_m[0, q))[lo, lo + cnt)

constexpr int kMergeE = 8;  // outputs per thread

template <typename T>
__global__ void merge_kernel(const T* __restrict__ A, Addr aa, int p, const T* __restrict__ B,
                             Addr ab, int q, T* __restrict__ O, Addr ao, int lo, int cnt,
                             long problems) {
  const long per = (cnt + kMergeE - 1) / kMergeE;
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= problems * per) return;
  const long m = gid / per;
  const int o0 = (int)(gid - m * per) * kMergeE;
  const T* a = A + aa.at(m);
  const T* b = B + ab.at(m);
  T* o = O + ao.at(m);
  const int d = lo + o0;  // absolute rank of the first output
  // merge path: smallest i with a[i] > b[d - i - 1] ... ties to A
  int i_lo = d - q > 0 ? d - q : 0, i_hi = d < p ? d : p;
  while (i_lo < i_hi) {
    const int i = (i_lo + i_hi) >> 1;
    const int j = d - i;
    // take i+1 from A if a[i] <= b[j-1]
    if (j > 0 && i < p && a[i] <= b[j - 1]) i_lo = i + 1;
    else i_hi = i;
  }
  int i = i_lo, j = d - i_lo;
  const int end = min(cnt, o0 + kMergeE);
  for (int t = o0; t < end; t++) {
    T v;
    if (j >= q || (i < p && a[i] <= b[j])) v = a[i++];
    else v = b[j++];
    o[t] = v;
  }
}

template <typename T>
static void merge(const T* A, Addr aa, int p, const T* B, Addr ab, int q, T* O, Addr ao, int lo,
                  int cnt, long problems, cudaStream_t s) {
  if (problems <= 0 || cnt <= 0) return;
  const long per = (cnt + kMergeE - 1) / kMergeE;
  const long threads = problems * per;
  const int bs = 256;
  merge_kernel<T><<<(unsigned)((threads + bs - 1) / bs), bs, 0, s>>>(A, aa, p, B, ab, q, O, ao,
                                                                     lo, cnt, problems);
}

// ------------------------------------------------------------------------
// run construction: gather `len` image samples per run and sort them.

enum GatherMode : int {
  kRows = 0,     // run (cx, j):  img[y_lo + j][clamp(cx*t + t-1-h + i)]
  kCols = 1,     // run (cy, x):  img[clamp(py0 + cy*t + t-1-h + i)][x]
  kRowExt = 2,   // run (cxc, j): img[y_lo + j][gx(cxc, i)]   (corner packs)
  kColExt = 3,   // run (cyc, x): img[gy(cyc, i)][x]
};

struct Gather {
  int mode;
  int len;
  int t;       // tile side (init) or parent side s (ext)
  int h;       // k / 2
  int c;       // parent core size (ext)
  int y_lo;    // first buffered image row
  int py0;     // first output row of the band (image coords)
  int n_inner; // runs per outer index (n_y for rows, W for cols)
  int W, H;
};

template <typename T>
__device__ __forceinline__ T gather_at(const Job& job, const Gather& g, long run, int i) {
  const long outer = run / g.n_inner;
  const int inner = (int)(run - outer * g.n_inner);
  int y, x;
  switch (g.mode) {
    case kRows:
      y = g.y_lo + inner;
      x = clampi((int)outer * g.t + g.t - 1 - g.h + i, 0, g.W - 1);
      break;
    case kCols:
      y = clampi(g.py0 + (int)outer * g.t + g.t - 1 - g.h + i, 0, g.H - 1);
      x = inner;
      break;
    case kRowExt: {
      const int cxc = (int)outer;
      const int pcx = (cxc >> 1) * g.t + g.t - 1 - g.h;
      const int gx0 = (cxc & 1) ? pcx + g.c : pcx - g.len;
      y = g.y_lo + inner;
      x = clampi(gx0 + i, 0, g.W - 1);
      break;
    }
    default: {
      const int cyc = (int)outer;
      const int pcy = g.py0 + (cyc >> 1) * g.t + g.t - 1 - g.h;
      const int gy0 = (cyc & 1) ? pcy + g.c : pcy - g.len;
      y = clampi(gy0 + i, 0, g.H - 1);
      x = inner;
      break;
    }
  }
  return load_px<T>(job, y, x);
}

template <int N>
__device__ __forceinline__ void sort_net(uint32_t (&v)[N]) {
  // Batcher odd-even merge sort on N = 2^m registers (fully unrolled)
#pragma unroll
  for (int p = 1; p < N; p <<= 1) {
#pragma unroll
    for (int k = p; k >= 1; k >>= 1) {
#pragma unroll
      for (int j = k % p; j + k < N; j += 2 * k) {
#pragma unroll
        for (int i = 0; i < k; i++) {
          if (i + j + k < N && (i + j) / (2 * p) == (i + j + k) / (2 * p)) {
            const uint32_t a = v[i + j], b = v[i + j + k];
            v[i + j] = min(a, b);
            v[i + j + k] = max(a, b);
          }
        }
      }
    }
  }
}

template <typename T, int P>
__global__ void __launch_bounds__(128) sort_runs_kernel(Job job, Gather g, T* __restrict__ out,
                                                        long runs) {
  const long run = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (run >= runs) return;
  uint32_t v[P];
#pragma unroll
  for (int i = 0; i < P; i++) v[i] = i < g.len ? (uint32_t)gather_at<T>(job, g, run, i) : 0xFFFFFFFFu;
  sort_net<P>(v);
  T* o = out + run * g.len;
#pragma unroll
  for (int i = 0; i < P; i++)
    if (i < g.len) o[i] = (T)v[i];
}

template <typename T>
static int sort_runs(const Job& job, const Gather& g, T* out, long runs, cudaStream_t s) {
  if (runs <= 0) return 0;
  const int bs = 128;
  const unsigned grid = (unsigned)((runs + bs - 1) / bs);
  if (g.len <= 1) sort_runs_kernel<T, 1><<<grid, bs, 0, s>>>(job, g, out, runs);
  else if (g.len <= 2) sort_runs_kernel<T, 2><<<grid, bs, 0, s>>>(job, g, out, runs);
  else if (g.len <= 4) sort_runs_kernel<T, 4><<<grid, bs, 0, s>>>(job, g, out, runs);
  else if (g.len <= 8) sort_runs_kernel<T, 8><<<grid, bs, 0, s>>>(job, g, out, runs);
  else if (g.len <= 16) sort_runs_kernel<T, 16><<<grid, bs, 0, s>>>(job, g, out, runs);
  else if (g.len <= 32) sort_runs_kernel<T, 32><<<grid, bs, 0, s>>>(job, g, out, runs);
  else if (g.len <= 64) sort_runs_kernel<T, 64><<<grid, bs, 0, s>>>(job, g, out, runs);
  else if (g.len <= 128) sort_runs_kernel<T, 128><<<grid, bs, 0, s>>>(job, g, out, runs);
  else return -1;
  return 0;
}

// ------------------------------------------------------------------------
// gather runs of a buffer into contiguous problem blocks (pack round 0)
//   dst[m][r][i] = src[row_of(m, r)][i],  row_of via a small mode switch

enum PackMode : int {
  kPackCols = 0,  // m = cy*(2n_cx) + cxc; runs cols[cy][gx(cxc, r)]      (len c)
  kPackRows = 1,  // m = cyc*(2n_cx) + cxc; runs rows2[cxc][gy(cyc,r)-y_lo] (len c2)
  kCoreRows = 2,  // m = cy*n_cx + cx;      runs rows[cx][rel(cy, r)]       (len c)
};

struct PackSpec {
  int mode, runs, len;
  int n_cx2;     // problems per outer row (2*n_cx or n_cx)
  int s, h, c;   // parent side, k/2, parent core
  int W, H, y_lo, py0, n_y;
};

template <typename T>
__global__ void pack_gather_kernel(const T* __restrict__ src, PackSpec ps, T* __restrict__ dst,
                                   long total) {
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= total) return;
  const int i = (int)(gid % ps.len);
  const long mr = gid / ps.len;
  const int r = (int)(mr % ps.runs);
  const long m = mr / ps.runs;
  const int outer = (int)(m / ps.n_cx2), inner = (int)(m % ps.n_cx2);
  long row;
  if (ps.mode == kPackCols) {
    const int cy = outer, cxc = inner;
    const int pcx = (cxc >> 1) * ps.s + ps.s - 1 - ps.h;
    const int gx0 = (cxc & 1) ? pcx + ps.c : pcx - ps.runs;
    const int x = clampi(gx0 + r, 0, ps.W - 1);
    row = (long)cy * ps.W + x;
  } else if (ps.mode == kPackRows) {
    const int cyc = outer, cxc = inner;
    const int pcy = ps.py0 + (cyc >> 1) * ps.s + ps.s - 1 - ps.h;
    const int gy0 = (cyc & 1) ? pcy + ps.c : pcy - ps.runs;
    const int y = clampi(gy0 + r, 0, ps.H - 1) - ps.y_lo;
    row = (long)cxc * ps.n_y + y;
  } else {
    const int cy = outer, cx = inner;
    const int y = clampi(ps.py0 + cy * ps.s + ps.s - 1 - ps.h + r, 0, ps.H - 1) - ps.y_lo;
    row = (long)cx * ps.n_y + y;
  }
  dst[gid] = src[row * ps.len + i];
}

// k-way merge of `runs` contiguous runs of `len` per problem (binary
// reduction, odd run carried), keeping [lo, lo + cnt) of the result.
template <typename T>
static void kway(T* buf, T* tmp, long problems, int runs, int len, T* out, int lo, int cnt,
                 cudaStream_t s) {
  // buf holds problems x runs x len; run r of problem m at m*runs*len + r*len
  const long block = (long)runs * len;
  std::vector<int> sizes(runs, len);
  T* cur = buf;
  T* nxt = tmp;
  while (sizes.size() > 1) {
    std::vector<int> ns;
    long off = 0, noff = 0;
    const bool last = sizes.size() == 2;
    for (size_t a = 0; a + 1 < sizes.size(); a += 2) {
      const int p = sizes[a], q = sizes[a + 1];
      if (last) {
        merge<T>(cur + off, lin(block), p, cur + off + p, lin(block), q, out, lin(cnt), lo, cnt,
                 problems, s);
      } else {
        merge<T>(cur + off, lin(block), p, cur + off + p, lin(block), q, nxt + noff, lin(block),
                 0, p + q, problems, s);
      }
      off += p + q;
      noff += p + q;
      ns.push_back(p + q);
    }
    if (sizes.size() % 2) {
      const int p = sizes.back();
      // carry the odd run: copy via a merge with an empty run
      merge<T>(cur + off, lin(block), p, cur + off, lin(block), 0, nxt + noff, lin(block), 0, p,
               problems, s);
      ns.push_back(p);
    }
    if (last) return;
    std::swap(cur, nxt);
    sizes = ns;
  }
  // single run: slice it
  merge<T>(cur, lin(block), sizes[0], cur, lin(block), 0, out, lin(cnt), lo, cnt, problems, s);
}

// ------------------------------------------------------------------------
// finalize: per pixel, rank q among cand (n) + col run (c) + row run (c) + corner

template <typename T>
__device__ __forceinline__ T kth4(const T* a, int na, const T* b, int nb, const T* c, int nc, T z,
                                  int q) {
  // q-th (0-based) smallest of the union of three sorted arrays and z.
  // Repeatedly discard a prefix of the array whose probe is smallest.
  int ia = 0, ib = 0, ic = 0, iz = 0;
  const T kMax = (T)~(T)0;
  while (true) {
    const int ra = na - ia, rb = nb - ib, rc = nc - ic, rz = 1 - iz;
    int alive = (ra > 0) + (rb > 0) + (rc > 0) + (rz > 0);
    if (q == 0 || alive == 1) {
      T best = kMax;
      bool any = false;
      // with alive == 1 the answer is at offset q of the surviving array
      if (alive == 1) {
        if (ra > 0) return a[ia + q];
        if (rb > 0) return b[ib + q];
        if (rc > 0) return c[ic + q];
        return z;
      }
      if (ra > 0) { best = a[ia]; any = true; }
      if (rb > 0 && (!any || b[ib] < best)) { best = b[ib]; any = true; }
      if (rc > 0 && (!any || c[ic] < best)) { best = c[ic]; any = true; }
      if (rz > 0 && (!any || z < best)) { best = z; }
      return best;
    }
    int step = (q + 1) / alive;
    if (step < 1) step = 1;
    const int sa = min(step, ra), sb = min(step, rb), sc = min(step, rc), sz = min(step, rz);
    // probes: the last element each array would give up
    T pa = sa ? a[ia + sa - 1] : kMax;
    T pb = sb ? b[ib + sb - 1] : kMax;
    T pc = sc ? c[ic + sc - 1] : kMax;
    T pz = sz ? z : kMax;
    int which = -1;
    T best = kMax;
    if (sa && (which < 0 || pa < best)) { which = 0; best = pa; }
    if (sb && (which < 0 || pb < best)) { which = 1; best = pb; }
    if (sc && (which < 0 || pc < best)) { which = 2; best = pc; }
    if (sz && (which < 0 || pz < best)) { which = 3; best = pz; }
    // the smallest probe and everything before it rank below q: drop them
    if (which == 0) { ia += sa; q -= sa; }
    else if (which == 1) { ib += sb; q -= sb; }
    else if (which == 2) { ic += sc; q -= sc; }
    else { iz += sz; q -= sz; }
  }
}

template <typename T>
__global__ void finalize_kernel(Job job, const T* __restrict__ cand, int n_cand,
                                const T* __restrict__ cols, const T* __restrict__ rows, int c,
                                int k, int d_lo, int py0, int band_h, int y_lo, int n_y,
                                int n_cx) {
  const int px = blockIdx.x * blockDim.x + threadIdx.x;
  const int ly = blockIdx.y;  // row within the band
  const int W = job.width;
  if (px >= W || ly >= band_h) return;
  const int h = k / 2;
  const int py = py0 + ly;  // image row
  const int lpy = py - job.out_y0;
  const int xg = clampi((px & 1) ? px + h : px - h, 0, W - 1);
  const int yg = clampi((lpy & 1) ? py + h : py - h, 0, job.src_h - 1);
  const int cy = ly >> 1, cx = px >> 1;
  const T* cd = cand + ((long)cy * n_cx + cx) * n_cand;
  const T* cr = cols + ((long)cy * W + xg) * c;
  const T* rr = rows + ((long)cx * n_y + (yg - y_lo)) * c;
  const T z = load_px<T>(job, yg, xg);
  const int q = (k * k + 1) / 2 - 1 - d_lo;
  const T v = kth4<T>(cd, n_cand, cr, c, rr, c, z, q);
  store_px<T>(job, lpy, px, v);
}

// ------------------------------------------------------------------------
// host driver

// The pass buffers come from a private stream-ordered pool per device: freed
// buffers stay reserved between calls (up to kKeepBytes) without changing the
// release threshold of the device's default pool, which other users of
// cudaMallocAsync in the process (e.g. PyTorch) rely on.
inline cudaMemPool_t pass_pool() {
  constexpr int kMaxDev = 64;
  constexpr uint64_t kKeepBytes = 1ull << 30;
  static std::mutex mu;
  static cudaMemPool_t pools[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
      cudaGetLastError();
      pools[dev] = nullptr;
      return nullptr;
    }
    uint64_t thr = kKeepBytes;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return pools[dev];
}

template <typename T>
struct Arena {
  cudaStream_t s;
  cudaMemPool_t pool = pass_pool();
  std::vector<void*> ptrs;
  T* get(long n) {
    void* p = nullptr;
    const size_t bytes = (size_t)std::max(n, 1L) * sizeof(T);
    const cudaError_t e = pool ? cudaMallocFromPoolAsync(&p, bytes, pool, s)
                               : cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  void release(T* p) {
    for (auto& q : ptrs)
      if (q == p) {
        cudaFreeAsync(q, s);
        q = nullptr;
      }
  }
  ~Arena() {
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, s);
  }
};

// Bytes of the largest level of a band of `br` root-tile rows (aware.py:416-434).
inline long peak_bytes(int k, int t, int W, int br, int esz) {
  const long Hb = (long)br * t;
  long n_cx = (W + t - 1) / t, n_cy = br;
  const long n_y = Hb + k;
  long peak = 0;
  for (int s = t; s >= 2; s /= 2) {
    const int c = k - s + 1;
    const Win w = retention((long)k * k, (long)c * c);
    long lvl = n_cx * n_y * c + n_cy * W * c + n_cy * n_cx * (w.hi - w.lo + 1);
    // our passes keep parent + child buffers alive and pack temporaries
    lvl = lvl * 3;
    peak = std::max(peak, lvl);
    n_cx *= 2;
    n_cy *= 2;
  }
  return peak * esz;
}

template <typename T>
static int run_band(const Job& job, int k, int t, int ty0, int ty1, cudaStream_t s) {
  Arena<T> ar{s, {}};
  const int W = job.width, H = job.src_h, h = k / 2;
  const long n_total = (long)k * k;
  int c = k - t + 1;
  const int n_tx = (W + t - 1) / t;
  int n_cy = ty1 - ty0;
  const int py0 = job.out_y0 + ty0 * t;
  const int y_lo = std::max(0, py0 - h);
  const int y_hi = std::min(H - 1, py0 + n_cy * t - 1 + h);
  const int n_y = y_hi - y_lo + 1;
  int n_cx = n_tx;

  // ---- pass_init ---------------------------------------------------------
  T* rows = ar.get((long)n_cx * n_y * c);
  T* cols = ar.get((long)n_cy * W * c);
  if (!rows || !cols) return (int)cudaErrorMemoryAllocation;
  Gather g{kRows, c, t, h, c, y_lo, py0, n_y, W, H};
  if (sort_runs<T>(job, g, rows, (long)n_cx * n_y, s)) return (int)cudaErrorInvalidValue;
  g.mode = kCols;
  g.n_inner = W;
  if (sort_runs<T>(job, g, cols, (long)n_cy * W, s)) return (int)cudaErrorInvalidValue;
  Win w = retention(n_total, (long)c * c);
  int n_cand = w.hi - w.lo + 1;
  int d_lo = w.lo - 1;
  T* cand = ar.get((long)n_cy * n_cx * n_cand);
  {
    const long problems = (long)n_cy * n_cx;
    T* blk = ar.get(problems * c * c);
    T* tmp = ar.get(problems * c * c);
    if (!cand || !blk || !tmp) return (int)cudaErrorMemoryAllocation;
    PackSpec ps{kCoreRows, c, c, n_cx, t, h, c, W, H, y_lo, py0, n_y};
    const long total = problems * c * c;
    pack_gather_kernel<T><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(rows, ps, blk, total);
    kway<T>(blk, tmp, problems, c, c, cand, w.lo - 1, n_cand, s);
    ar.release(blk);
    ar.release(tmp);
  }

  // ---- pass_extend_level: fused H + V split until 2x2 tiles --------------
  int side = t;
  while (side > 2) {
    const int gg = side / 2, c2 = c + gg;
    const long np_h = (long)n_cy * 2 * n_cx;
    // horizontal absorb: pack the gained column runs, merge, trim
    T* pk = ar.get(np_h * gg * c);
    T* tmp = ar.get(np_h * gg * c);
    T* packh = ar.get(np_h * gg * c);
    if (!pk || !tmp || !packh) return (int)cudaErrorMemoryAllocation;
    {
      PackSpec ps{kPackCols, gg, c, 2 * n_cx, side, h, c, W, H, y_lo, py0, n_y};
      const long total = np_h * gg * c;
      pack_gather_kernel<T><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(cols, ps, pk, total);
      kway<T>(pk, tmp, np_h, gg, c, packh, 0, gg * c, s);
    }
    ar.release(pk);
    ar.release(tmp);
    Win wh = retention(n_total, (long)c2 * c);
    const int lo_h = wh.lo - 1 - d_lo, cnt_h = wh.hi - wh.lo + 1;
    T* candh = ar.get(np_h * cnt_h);
    if (!candh) return (int)cudaErrorMemoryAllocation;
    // cand (n_cy, n_cx, n_cand) parent of child (cy, cxc) is (cy, cxc/2)
    merge<T>(cand, Addr{(long)n_cx * n_cand, n_cand, 2 * n_cx, 0, 1}, n_cand, packh,
             lin((long)gg * c), gg * c, candh, lin(cnt_h), lo_h, cnt_h, np_h, s);
    ar.release(packh);
    ar.release(cand);
    d_lo = wh.lo - 1;
    // row extension: corner packs widen every run to the child core width
    const long nrun_r = (long)2 * n_cx * n_y;
    T* ext = ar.get(nrun_r * gg);
    T* rows2 = ar.get(nrun_r * c2);
    if (!ext || !rows2) return (int)cudaErrorMemoryAllocation;
    {
      Gather ge{kRowExt, gg, side, h, c, y_lo, py0, n_y, W, H};
      if (sort_runs<T>(job, ge, ext, nrun_r, s)) return (int)cudaErrorInvalidValue;
      // parent run of (cxc, j) is rows[cxc/2][j]
      // m = cxc*n_y + j -> parent (cxc/2)*n_y*c + j*c
      merge<T>(rows, Addr{(long)n_y * c, c, n_y, 1, 0}, c, ext, lin(gg), gg, rows2,
               lin(c2), 0, c2, nrun_r, s);
    }
    ar.release(ext);
    ar.release(rows);
    rows = rows2;
    // vertical absorb: gained rows arrive already extended
    const long np_v = (long)2 * n_cy * 2 * n_cx;
    T* pk2 = ar.get(np_v * gg * c2);
    T* tmp2 = ar.get(np_v * gg * c2);
    T* packv = ar.get(np_v * gg * c2);
    if (!pk2 || !tmp2 || !packv) return (int)cudaErrorMemoryAllocation;
    {
      PackSpec ps{kPackRows, gg, c2, 2 * n_cx, side, h, c, W, H, y_lo, py0, n_y};
      const long total = np_v * gg * c2;
      pack_gather_kernel<T><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(rows, ps, pk2, total);
      kway<T>(pk2, tmp2, np_v, gg, c2, packv, 0, gg * c2, s);
    }
    ar.release(pk2);
    ar.release(tmp2);
    Win wv = retention(n_total, (long)c2 * c2);
    const int lo_v = wv.lo - 1 - d_lo, cnt_v = wv.hi - wv.lo + 1;
    T* cand2 = ar.get(np_v * cnt_v);
    if (!cand2) return (int)cudaErrorMemoryAllocation;
    // child (cyc, cxc) takes candh[cyc/2][cxc]: m = cyc*(2n_cx) + cxc
    merge<T>(candh, Addr{(long)2 * n_cx * cnt_h, cnt_h, 2 * n_cx, 1, 0}, cnt_h, packv,
             lin((long)gg * c2), gg * c2, cand2, lin(cnt_v), lo_v, cnt_v, np_v, s);
    ar.release(packv);
    ar.release(candh);
    cand = cand2;
    n_cand = cnt_v;
    d_lo = wv.lo - 1;
    // column extension for the next level
    const long nrun_c = (long)2 * n_cy * W;
    T* extc = ar.get(nrun_c * gg);
    T* cols2 = ar.get(nrun_c * c2);
    if (!extc || !cols2) return (int)cudaErrorMemoryAllocation;
    {
      Gather ge{kColExt, gg, side, h, c, y_lo, py0, W, W, H};
      if (sort_runs<T>(job, ge, extc, nrun_c, s)) return (int)cudaErrorInvalidValue;
      // parent of (cyc, x) is cols[cyc/2][x]: m = cyc*W + x
      merge<T>(cols, Addr{(long)W * c, c, W, 1, 0}, c, extc, lin(gg), gg, cols2, lin(c2), 0,
               c2, nrun_c, s);
    }
    ar.release(extc);
    ar.release(cols);
    cols = cols2;
    n_cy *= 2;
    n_cx *= 2;
    c = c2;
    side = gg;
  }

  // ---- pass_finalize -----------------------------------------------------
  const int band_h = std::min(n_cy * 2, job.out_y0 + job.out_h - py0);
  dim3 grid((W + 127) / 128, band_h);
  finalize_kernel<T><<<grid, 128, 0, s>>>(job, cand, n_cand, cols, rows, c, k, d_lo, py0, band_h,
                                          y_lo, n_y, n_cx);
  return (int)cudaGetLastError();
}

template <typename T>
static int launch_t(const Job& job0, int k, cudaStream_t s, long budget) {
  const int t = root_tile(k);
  const int n_ty = (job0.out_h + t - 1) / t;
  int br = n_ty;
  while (br > 1 && peak_bytes(k, t, job0.width, br, sizeof(T)) > budget) br = (br + 1) / 2;
  for (int c = 0; c < job0.channels; c++) {
    Job job = job0;
    job.src = static_cast<const T*>(job0.src) + c;
    job.dst = static_cast<T*>(job0.dst) + c;
    job.src_pitch = job0.src_pitch;
    // per-channel view: x stride = channels, handled by load_px/store_px with
    // blockIdx.z == 0 -- fold the channel into the base pointer instead
    for (int a = 0; a < n_ty; a += br) {
      const int rc = run_band<T>(job, k, t, a, std::min(a + br, n_ty), s);
      if (rc) return rc;
    }
  }
  return 0;
}

}  // namespace aware

int launch_aware(int bits, const Job& job, int k, cudaStream_t s) {
  const long budget = 3L << 30;  // device bytes per band
  switch (bits) {
    case 8: return aware::launch_t<uint8_t>(job, k, s, budget);
    case 16: return aware::launch_t<uint16_t>(job, k, s, budget);
    default: return aware::launch_t<uint32_t>(job, k, s, budget);
  }
}

}  // namespace tmb
