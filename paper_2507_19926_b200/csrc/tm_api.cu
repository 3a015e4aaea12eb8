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

// Kernel routing.  Results are identical whichever exact kernel runs; the
// variant only chooses the algorithm (engine.py:36-52).
bool supports(int kernel, int bits, int kw, int kh) {
  const bool square = kw == kh;
  switch (kernel) {
    case TM_KERNEL_OBLIVIOUS: return square && find_obl(bits, kw) != nullptr;
    case TM_KERNEL_MULTIPASS: return square && kw >= 9;
    case TM_KERNEL_SELECT: return true;
    case TM_KERNEL_HISTOGRAM: return square && bits == 8 && tmb::hist8_supports(kw);
    case TM_KERNEL_RANK: return square && tmb::rank_supports(bits, kw);
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
// .jsonl): the oblivious network up to the crossover, the data-aware kernel
// from it on.  Crossovers: 8-bit k = 15, 16-bit k = 27, 32-bit k = 23.
int auto_kernel(int bits, int k) {
  if (k == 3) return TM_KERNEL_MED3;
  const int crossover = bits == 8 ? 15 : (bits == 16 ? 27 : 23);
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
      return square ? auto_kernel(bits, kw) : TM_KERNEL_SELECT;
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
  int err;
  switch (route(bits, k_w, k_h, variant)) {
    case TM_KERNEL_OBLIVIOUS:
      err = find_obl(bits, k_w)->fn(job, s);
      break;
    case TM_KERNEL_MULTIPASS:
      err = tmb::launch_aware(bits, job, k_w, s);
      break;
    case TM_KERNEL_HISTOGRAM:
      err = tmb::launch_hist8(job, k_w, s);
      break;
    case TM_KERNEL_RANK:
      err = tmb::launch_rank(bits, job, k_w, s);
      break;
    case TM_KERNEL_MED3:
      err = tmb::launch_med3(bits, job, s);
      break;
    default:
      err = tmb::launch_select(bits, job, k_w, k_h, s);
      break;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (err != cudaSuccess)
    return fail(TM_ECUDA, "CUDA launch failed: %s", cudaGetErrorString((cudaError_t)err));
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

int tm_median2d_host(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                     int32_t width, int32_t height, int32_t channels, int32_t bits, int32_t k_w,
                     int32_t k_h, int32_t variant, int32_t device) {
  int rc = check_common(width, height, bits, k_w, k_h, variant);
  if (rc) return rc;
  if (!src || !dst) return fail(TM_EINVAL, "null buffer");
  if (channels < 1) return fail(TM_EINVAL, "bad channel count %d", channels);
  const int64_t row = (int64_t)width * channels * (bits / 8);
  if (src_pitch < row || dst_pitch < row) return fail(TM_EINVAL, "pitch smaller than a row");
  // Row bands pipelined over streams: band b's H2D copy, the filters of
  // earlier bands (three filter streams, so band kernels overlap each other's
  // tails) and their D2H copies run concurrently (PCIe is full duplex), so the
  // call costs about max(H2D, filter, D2H) instead of their sum.  A band's
  // filter waits for the input chunk holding its last halo row.
  constexpr int kMaxBands = 32;
  constexpr int kFilterStreams = 3;  // band kernels overlap each other's tails
  struct Scratch {
    void* buf = nullptr;
    size_t bytes = 0;
    cudaStream_t st[3] = {nullptr, nullptr, nullptr};  // h2d, filter, d2h
    cudaStream_t fs[kFilterStreams] = {};               // concurrent band filters
    cudaEvent_t ev_in[kMaxBands] = {}, ev_out[kMaxBands] = {};
  };
  static thread_local std::vector<Scratch> per_dev;
  if (device < 0) return fail(TM_EINVAL, "bad device %d", device);
  if ((int)per_dev.size() <= device) per_dev.resize(device + 1);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(TM_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  Scratch& sc = per_dev[device];
  const size_t need = 2 * (size_t)row * height;
  if (sc.bytes < need) {
    if (sc.buf) cudaFree(sc.buf);
    sc.buf = nullptr;
    sc.bytes = 0;
    e = cudaMalloc(&sc.buf, need);
    if (e != cudaSuccess) return fail(TM_ECUDA, "cudaMalloc: %s", cudaGetErrorString(e));
    sc.bytes = need;
  }
  if (!sc.st[0]) {
    for (auto& st : sc.st) {
      e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      if (e != cudaSuccess) return fail(TM_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    for (auto& st : sc.fs) {
      e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      if (e != cudaSuccess) return fail(TM_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    for (int b = 0; b < kMaxBands; b++) {
      e = cudaEventCreateWithFlags(&sc.ev_in[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sc.ev_out[b], cudaEventDisableTiming);
      if (e != cudaSuccess) return fail(TM_ECUDA, "cudaEventCreate: %s", cudaGetErrorString(e));
    }
  }
  char* din = static_cast<char*>(sc.buf);
  char* dout = din + (size_t)row * height;
  const int halo = k_h / 2;
  // bands of >= 64 rows and >= 2 MB, at most 16 (measured on C2: 1 -> 19.3,
  // 4 -> 27.8, 8 -> 34.7, 16 -> 38.7, 32 -> 35.5 Gpixel/s e2e); small images
  // get one band -- the pipeline only pays once copies dominate
  const int64_t img_bytes = row * height;
  static const int force_nb = [] {  // experiments: TMB_HOST_BANDS
    const char* v = getenv("TMB_HOST_BANDS");
    return v ? atoi(v) : 0;
  }();
  const int nb = force_nb > 0 ? std::min(std::min(force_nb, kMaxBands), height)
                              : (int)std::max<int64_t>(1, std::min<int64_t>(
                                    {16, height / 64, img_bytes / (2 << 20)}));
  int y[kMaxBands + 1];
  for (int b = 0; b <= nb; b++) y[b] = (int)((int64_t)height * b / nb);
  const char* hsrc = static_cast<const char*>(src);
  char* hdst = static_cast<char*>(dst);
  for (int b = 0; b < nb; b++) {
    const size_t n_rows = (size_t)(y[b + 1] - y[b]);
    e = src_pitch == row
            ? cudaMemcpyAsync(din + (size_t)y[b] * row, hsrc + (int64_t)y[b] * src_pitch,
                              n_rows * row, cudaMemcpyHostToDevice, sc.st[0])
            : cudaMemcpy2DAsync(din + (size_t)y[b] * row, row, hsrc + (int64_t)y[b] * src_pitch,
                                src_pitch, row, n_rows, cudaMemcpyHostToDevice, sc.st[0]);
    if (e == cudaSuccess) e = cudaEventRecord(sc.ev_in[b], sc.st[0]);
    if (e != cudaSuccess) return fail(TM_ECUDA, "H2D copy: %s", cudaGetErrorString(e));
  }
  for (int b = 0; b < nb; b++) {
    cudaStream_t fst = sc.fs[b % kFilterStreams];
    const int last_src = std::min(height, y[b + 1] + halo) - 1;
    int chunk = b;
    while (chunk + 1 < nb && y[chunk + 1] <= last_src) chunk++;
    e = cudaStreamWaitEvent(fst, sc.ev_in[chunk], 0);
    if (e != cudaSuccess) return fail(TM_ECUDA, "stream wait: %s", cudaGetErrorString(e));
    rc = tm_median2d_band(din, row, height, y[b], y[b + 1] - y[b], dout + (size_t)y[b] * row, row,
                          width, channels, bits, k_w, k_h, variant, fst);
    if (rc) return rc;
    e = cudaEventRecord(sc.ev_out[b], fst);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sc.st[2], sc.ev_out[b], 0);
    if (e == cudaSuccess)
      e = dst_pitch == row
              ? cudaMemcpyAsync(hdst + (int64_t)y[b] * dst_pitch, dout + (size_t)y[b] * row,
                                (size_t)(y[b + 1] - y[b]) * row, cudaMemcpyDeviceToHost, sc.st[2])
              : cudaMemcpy2DAsync(hdst + (int64_t)y[b] * dst_pitch, dst_pitch,
                                  dout + (size_t)y[b] * row, row, row, y[b + 1] - y[b],
                                  cudaMemcpyDeviceToHost, sc.st[2]);
    if (e != cudaSuccess) return fail(TM_ECUDA, "D2H copy: %s", cudaGetErrorString(e));
  }
  e = cudaStreamSynchronize(sc.st[2]);
  for (auto& st : sc.fs)
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sc.st[0]);
  if (e != cudaSuccess) return fail(TM_ECUDA, "kernel failed: %s", cudaGetErrorString(e));
  return TM_OK;
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
