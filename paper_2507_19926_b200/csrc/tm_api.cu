// tm_api.cu -- the C ABI (include/tilemedian_b200.h): validation, dispatch,
// launch accounting and the host-buffer entry point.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/tilemedian_b200.h"
#include "tm_kernels.h"

namespace tmb {
#include "gen/dispatch.inc"
}

namespace {

thread_local char g_err[512] = "";
thread_local int g_force = 0;
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

const tmb::OblEntry* find_obl(int bits, int k) {
  for (const auto& e : tmb::kOblTable)
    if (e.bits == bits && e.k == k) return &e;
  return nullptr;
}

int launch(int kernel, int bits, int k_w, int k_h, const tmb::Job& job, cudaStream_t s) {
  switch (kernel) {
    case TM_KERNEL_OBLIVIOUS: return find_obl(bits, k_w)->fn(job, s);
    case TM_KERNEL_MULTIPASS: return tmb::launch_aware(bits, job, k_w, s);
    case TM_KERNEL_HISTOGRAM:
      return k_w == k_h ? tmb::launch_hist8(job, k_w, s) : tmb::launch_hist8_rect(job, k_w, k_h, s);
    case TM_KERNEL_RANK:
      return k_w == k_h ? tmb::launch_rank(bits, job, k_w, s)
                        : tmb::launch_rank_rect(bits, job, k_w, k_h, s);
    case TM_KERNEL_MED3: return tmb::launch_med3(bits, job, s);
    default: return tmb::launch_select(bits, job, k_w, k_h, s);
  }
}

// Kernel routing.  Results are identical whichever exact kernel runs; the
// variant only chooses the algorithm (engine.py:36-52).
bool supports(int kernel, int bits, int kw, int kh) {
  const bool square = kw == kh;
  switch (kernel) {
    case TM_KERNEL_OBLIVIOUS: return square && find_obl(bits, kw) != nullptr;
    case TM_KERNEL_MULTIPASS: return square && kw >= 9;
    case TM_KERNEL_SELECT: return true;
    case TM_KERNEL_HISTOGRAM:
      return bits == 8 && (square ? tmb::hist8_supports(kw) : tmb::hist8_rect_supports(kw, kh));
    case TM_KERNEL_RANK:
      return square ? tmb::rank_supports(bits, kw) : tmb::rank_rect_supports(bits, kw, kh);
    case TM_KERNEL_MED3: return square && kw == 3;
    default: return false;
  }
}

// The data-aware kernel for (bits, k): sliding histograms of the samples for
// 8-bit data, of 7-bit keys (coarse + candidate passes) for 16/32-bit data.
int aware_kernel(int bits, int k) {
  if (bits == 8 && tmb::hist8_supports(k)) return TM_KERNEL_HISTOGRAM;
  if (tmb::rank_supports(bits, k)) return TM_KERNEL_RANK;
  return TM_KERNEL_MULTIPASS;
}

// "auto": the fastest exact kernel per (bits, k), measured on B200 over the
// full k = 3..75 sweep of 4096^2 images (profiles/r01_sweep_4096_all_kernels
// .jsonl, re-measured in round 2 around the crossovers): the oblivious network
// up to the crossover, the data-aware kernel from it on.  Crossovers: 8-bit
// k = 13 (round 2: histogram 64.0 vs network 62.5 Gpx/s at 4096^2, 68.7 vs
// 64.4 at 8192^2), 16-bit k = 27, 32-bit k = 23.
int auto_kernel(int bits, int k) {
  if (k == 3) return TM_KERNEL_MED3;
  const int crossover = bits == 8 ? 13 : (bits == 16 ? 27 : 23);
  if (k < crossover && find_obl(bits, k)) return TM_KERNEL_OBLIVIOUS;
  return aware_kernel(bits, k);
}

int route(int bits, int kw, int kh, int variant) {
  if (g_force && supports(g_force, bits, kw, kh)) return g_force;
  const bool square = kw == kh;
  switch (variant) {
    case TM_VARIANT_ORACLE:
      return TM_KERNEL_SELECT;
    case TM_VARIANT_OBLIVIOUS:
      if (square && kw == 3) return TM_KERNEL_MED3;  // the k = 3 network, specialised
      return (square && find_obl(bits, kw)) ? TM_KERNEL_OBLIVIOUS : TM_KERNEL_SELECT;
    case TM_VARIANT_AWARE:
      return (square && kw >= 9) ? aware_kernel(bits, kw) : TM_KERNEL_SELECT;
    default:  // auto
      if (square) return auto_kernel(bits, kw);
      // rectangular: the data-aware sweeps (8-bit histogram, 16/32-bit rank)
      // for windows of >= 81 samples, else the exact per-pixel selection
      if (kw * kh >= 81) {
        if (bits == 8 && tmb::hist8_rect_supports(kw, kh)) return TM_KERNEL_HISTOGRAM;
        if (bits != 8 && tmb::rank_rect_supports(bits, kw, kh)) return TM_KERNEL_RANK;
      }
      return TM_KERNEL_SELECT;
  }
}

int check_common(int width, int rows, int bits, int kw, int kh, int variant) {
  if (bits != 8 && bits != 16 && bits != 32)
    return fail(TM_ETYPE, "unsupported element width %d bits (expected 8, 16 or 32)", bits);
  if (width < 1 || rows < 1)
    return fail(TM_EINVAL, "expected a non-empty 2-D image, got %dx%d", width, rows);
  if (kw < 3 || kh < 3 || !(kw & 1) || !(kh & 1))
    return fail(TM_EINVAL, "kernel sides must be odd and >= 3, got %dx%d", kw, kh);
  if (kw > 127 || kh > 127)
    return fail(TM_EINVAL, "kernel sides above 127 are not supported, got %dx%d", kw, kh);
  if (variant < TM_VARIANT_AUTO || variant > TM_VARIANT_ORACLE)
    return fail(TM_EINVAL, "unknown variant %d", variant);
  return TM_OK;
}

}  // namespace

namespace tmb {
int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
}  // namespace tmb

extern "C" {

int tm_median2d_band(const void* src, int64_t src_pitch, int32_t src_rows, int32_t out_row0,
                     int32_t out_rows, void* dst, int64_t dst_pitch, int32_t width,
                     int32_t channels, int32_t bits, int32_t k_w, int32_t k_h,
                     int32_t variant, void* stream) {
  int rc = check_common(width, src_rows, bits, k_w, k_h, variant);
  if (rc) return rc;
  if (!src || !dst) return fail(TM_EINVAL, "null buffer");
  if (channels < 1 || channels > 65535) return fail(TM_EINVAL, "bad channel count %d", channels);
  const int esz = bits / 8;
  if (out_row0 < 0 || out_rows < 0 || out_row0 + out_rows > src_rows)
    return fail(TM_EINVAL, "output rows [%d, %d) outside source rows [0, %d)", out_row0,
                out_row0 + out_rows, src_rows);
  if (src_pitch % esz || dst_pitch % esz)
    return fail(TM_EINVAL, "pitches must be multiples of the element size");
  if (src_pitch < (int64_t)width * channels * esz || dst_pitch < (int64_t)width * channels * esz)
    return fail(TM_EINVAL, "pitch smaller than a row");
  if (out_rows == 0) return TM_OK;
  tmb::Job job;
  job.src = src;
  job.dst = dst;
  job.src_pitch = src_pitch / esz;
  job.dst_pitch = dst_pitch / esz;
  job.width = width;
  job.src_h = src_rows;
  job.out_y0 = out_row0;
  job.out_h = out_rows;
  job.channels = channels;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int kernel = route(bits, k_w, k_h, variant);
  // at most 65535 output rows per launch (grid.y of the row-tiled kernels);
  // taller images are launched in row chunks of the same source
  constexpr int kMaxLaunchRows = 65535;
  for (int r0 = 0; r0 < out_rows; r0 += kMaxLaunchRows) {
    tmb::Job part = job;
    part.out_y0 = out_row0 + r0;
    part.out_h = std::min(kMaxLaunchRows, out_rows - r0);
    part.dst = static_cast<char*>(dst) + (int64_t)r0 * dst_pitch;
    const int err = launch(kernel, bits, k_w, k_h, part, s);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (err != cudaSuccess)
      return fail(TM_ECUDA, "CUDA launch failed: %s", cudaGetErrorString((cudaError_t)err));
  }
  return TM_OK;
}

int tm_median2d_rect(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                     int32_t width, int32_t height, int32_t bits, int32_t k_w, int32_t k_h,
                     int32_t variant, void* stream) {
  return tm_median2d_band(src, src_pitch, height, 0, height, dst, dst_pitch, width, 1, bits, k_w,
                          k_h, variant, stream);
}

int tm_median2d(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch, int32_t width,
                int32_t height, int32_t bits, int32_t k, int32_t variant, void* stream) {
  return tm_median2d_band(src, src_pitch, height, 0, height, dst, dst_pitch, width, 1, bits, k, k,
                          variant, stream);
}

int tm_median2d_planes(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                       int32_t width, int32_t height, int32_t channels, int32_t bits, int32_t k,
                       int32_t variant, void* stream) {
  return tm_median2d_band(src, src_pitch, height, 0, height, dst, dst_pitch, width, channels, bits,
                          k, k, variant, stream);
}

int tm_dispatch_query(int32_t bits, int32_t k_w, int32_t k_h, int32_t variant) {
  if (check_common(1, 1, bits, k_w, k_h, variant)) return TM_KERNEL_NONE;
  return route(bits, k_w, k_h, variant);
}

const char* tm_kernel_name(int32_t kernel) {
  switch (kernel) {
    case TM_KERNEL_OBLIVIOUS: return "oblivious";
    case TM_KERNEL_MULTIPASS: return "multipass";
    case TM_KERNEL_SELECT: return "select";
    case TM_KERNEL_HISTOGRAM: return "histogram";
    case TM_KERNEL_RANK: return "rank";
    case TM_KERNEL_MED3: return "med3";
    default: return "none";
  }
}

int tm_force_kernel(int32_t kernel) {
  const int prev = g_force;
  g_force = kernel;
  return prev;
}

int64_t tm_launch_count(void) { return g_launches.load(); }

const char* tm_last_error(void) { return g_err; }

const char* tm_version(void) { return "tilemedian_b200 0.1.0 (sm_100a)"; }

}  // extern "C"
