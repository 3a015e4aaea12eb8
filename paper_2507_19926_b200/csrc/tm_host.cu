// tm_host.cu -- host-buffer entry points of the C ABI: the pipelined
// H2D -> filter -> D2H path for numpy images (tm_median2d_host), its
// multi-GPU row-band form (tm_median2d_host_multi), the device-resident
// multi-GPU band form with peer halo exchange (tm_median2d_bands), and the
// pinned host allocator the Python drop-in returns its outputs in.
//
// Reference role: filter_image / filter_planes on numpy arrays
// (engine.py:29-64) -- the reference works in host memory, so a drop-in call
// includes both copies -- and the reference's banding with re-read halos
// (aware.py:455-491), here one band per GPU.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/tilemedian_b200.h"
#include "tm_kernels.h"

namespace tmb {
int set_error(int code, const char* fmt, ...);  // tm_api.cu (thread-local message)
}

namespace {

using tmb::set_error;

// ---------------------------------------------------------------------------
// Restores the caller's current device on every return path.
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------------------
// Host copy workers.  Pageable <-> pinned staging copies run on a small pool
// of threads (one memcpy stream saturates well below the host's memory
// bandwidth); the caller participates.  One job at a time.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool p;
    return p;
  }
  // Calls fn(i) for i in [0, n), spread over the workers and the caller.
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 1 || workers_.empty()) {
      for (int i = 0; i < n; i++) fn(i);
      return;
    }
    std::lock_guard<std::mutex> one(run_mu_);
    Job job;
    job.fn = &fn;
    job.n = n;
    {
      std::lock_guard<std::mutex> g(mu_);
      cur_ = &job;
      gen_++;
    }
    cv_.notify_all();
    drain(job);
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return job.done == job.n && job.users == 0; });
    cur_ = nullptr;
  }
  // Row copy of `rows` rows of `row_bytes`, parallel over pieces of >= 256 KB.
  void copy2d(char* dst, int64_t dpitch, const char* src, int64_t spitch, int64_t row_bytes,
              int64_t rows) {
    if (rows <= 0) return;
    const int64_t total = row_bytes * rows;
    const int pieces = (int)std::max<int64_t>(1, std::min<int64_t>(2 * size(), total >> 18));
    const bool flat = dpitch == row_bytes && spitch == row_bytes;
    run(pieces, [&](int i) {
      if (flat) {
        const int64_t a = total * i / pieces, b = total * (i + 1) / pieces;
        std::memcpy(dst + a, src + a, (size_t)(b - a));
      } else {
        const int64_t a = rows * i / pieces, b = rows * (i + 1) / pieces;
        for (int64_t r = a; r < b; r++)
          std::memcpy(dst + r * dpitch, src + r * spitch, (size_t)row_bytes);
      }
    });
  }
  int size() const { return (int)workers_.size() + 1; }

 private:
  struct Job {
    const std::function<void(int)>* fn = nullptr;
    int n = 0;
    std::atomic<int> next{0};
    int done = 0;   // guarded by mu_
    int users = 0;  // workers inside drain(); guarded by mu_
  };
  CopyPool() {
    const char* env = getenv("TMB_COPY_THREADS");
    unsigned hw = std::thread::hardware_concurrency();
    // 8 by default: measured on the B200 box (16 vCPUs), 90 MB pageable input:
    // 1 thread 11.1 ms, 4: 4.5, 8: 4.4, 16: 5.5 per call (host memory bound)
    int n = env ? atoi(env) : (int)std::min(8u, hw > 1 ? hw : 1u);
    for (int i = 1; i < n; i++) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      Job* job;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || (gen_ != seen && cur_ != nullptr); });
        if (stop_) return;
        seen = gen_;
        job = cur_;
        job->users++;
      }
      drain(*job);
      std::lock_guard<std::mutex> g(mu_);
      if (--job->users == 0 && job->done == job->n) done_cv_.notify_all();
    }
  }
  void drain(Job& job) {
    for (;;) {
      const int i = job.next.fetch_add(1);
      if (i >= job.n) return;
      (*job.fn)(i);
      std::lock_guard<std::mutex> g(mu_);
      if (++job.done == job.n && job.users == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  Job* cur_ = nullptr;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// ---------------------------------------------------------------------------
// Pinned (page-locked, portable) host blocks, cached by size so repeated
// calls do not pay cudaHostAlloc.
class PinnedPool {
 public:
  static PinnedPool& get() {
    static PinnedPool p;
    return p;
  }
  void* alloc(size_t n) {
    n = std::max<size_t>(4096, (n + 4095) & ~(size_t)4095);
    {
      std::lock_guard<std::mutex> g(mu_);
      auto it = free_.lower_bound(n);
      if (it != free_.end() && it->first <= 2 * n) {
        void* p = it->second;
        cached_ -= it->first;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, n, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      trim(0);  // give cached blocks back and retry once
      if (cudaHostAlloc(&p, n, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
    }
    std::lock_guard<std::mutex> g(mu_);
    size_[p] = n;
    return p;
  }
  bool release(void* p) {
    if (!p) return true;
    std::lock_guard<std::mutex> g(mu_);
    auto it = size_.find(p);
    if (it == size_.end()) return false;
    free_.emplace(it->second, p);
    cached_ += it->second;
    trim_locked(kKeepBytes);
    return true;
  }
  void trim(size_t keep) {
    std::lock_guard<std::mutex> g(mu_);
    trim_locked(keep);
  }

 private:
  static constexpr size_t kKeepBytes = (size_t)4 << 30;  // cached, not in use
  void trim_locked(size_t keep) {
    while (cached_ > keep && !free_.empty()) {
      auto it = std::prev(free_.end());  // largest first
      cudaFreeHost(it->second);
      size_.erase(it->second);
      cached_ -= it->first;
      free_.erase(it);
    }
  }
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
  std::unordered_map<void*, size_t> size_;
  size_t cached_ = 0;
};

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// ---------------------------------------------------------------------------
// Per-device resources of the host path (process-wide, one call per device
// at a time).
constexpr int kMaxDev = 64;
constexpr int kMaxBands = 32;
constexpr int kFilterStreams = 3;  // band kernels overlap each other's tails

struct DevRes {
  std::mutex mu;
  bool init = false;
  void* dbuf = nullptr;  // device in + out
  size_t dbytes = 0;
  void* pin_in = nullptr;  // staging for pageable sources / destinations
  size_t pin_in_bytes = 0;
  void* pin_out = nullptr;
  size_t pin_out_bytes = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaStream_t fs[kFilterStreams] = {};
  cudaEvent_t ev_in[kMaxBands] = {}, ev_out[kMaxBands] = {}, ev_d2h[kMaxBands] = {};
};
DevRes g_dev[kMaxDev];

int ensure_init(DevRes& r) {
  if (r.init) return TM_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&r.h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.d2h, cudaStreamNonBlocking);
  for (auto& s : r.fs)
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int b = 0; b < kMaxBands && e == cudaSuccess; b++) {
    e = cudaEventCreateWithFlags(&r.ev_in[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.ev_out[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.ev_d2h[b], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return set_error(TM_ECUDA, "stream/event create: %s", cudaGetErrorString(e));
  r.init = true;
  return TM_OK;
}

int grow_device(DevRes& r, size_t need) {
  if (r.dbytes >= need) return TM_OK;
  if (r.dbuf) cudaFree(r.dbuf);
  r.dbuf = nullptr;
  r.dbytes = 0;
  cudaError_t e = cudaMalloc(&r.dbuf, need);
  if (e != cudaSuccess) return set_error(TM_ECUDA, "cudaMalloc(%zu): %s", need, cudaGetErrorString(e));
  r.dbytes = need;
  return TM_OK;
}

int grow_pinned(void*& p, size_t& have, size_t need) {
  if (have >= need) return TM_OK;
  PinnedPool::get().release(p);
  p = PinnedPool::get().alloc(need);
  have = p ? need : 0;
  if (!p) return set_error(TM_ECUDA, "pinned host allocation of %zu bytes failed", need);
  return TM_OK;
}

struct HostArgs {
  const char* src;
  int64_t src_pitch;
  char* dst;
  int64_t dst_pitch;
  int width, height, channels, bits, k_w, k_h, variant;
};

// Output rows [ya, yb) of the image in `a` on `device`: source rows
// [sa, sb) = [ya - h, yb + h) clamped go to the device, the band is filtered
// there (reads clamp only at the true image edges) and written back.  Inside,
// the band is split into up to 16 sub-bands pipelined over streams: H2D
// copies, filters (three streams, so band kernels overlap each other's tails)
// and D2H copies run concurrently (PCIe is full duplex).  A pageable source is
// staged into pinned memory by the copy workers a chunk ahead of its DMA; a
// pageable destination is drained from pinned memory as each D2H lands.
double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
const bool g_trace = [] {  // TMB_HOST_TRACE=1: per-call phase times on stderr
  const char* v = getenv("TMB_HOST_TRACE");
  return v && *v == '1';
}();

int host_chunk(const HostArgs& a, int device, int ya, int yb) {
  if (device < 0 || device >= kMaxDev) return set_error(TM_EINVAL, "bad device %d", device);
  DevRes& r = g_dev[device];
  std::lock_guard<std::mutex> lock(r.mu);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return set_error(TM_ECUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  int rc = ensure_init(r);
  if (rc) return rc;
  const int64_t row = (int64_t)a.width * a.channels * (a.bits / 8);
  const int halo = a.k_h / 2;
  const int sa = std::max(0, ya - halo), sb = std::min(a.height, yb + halo);
  const int src_rows = sb - sa, out_rows = yb - ya;
  rc = grow_device(r, (size_t)row * (src_rows + out_rows));
  if (rc) return rc;
  const bool stage_in = !is_pinned(a.src), stage_out = !is_pinned(a.dst);
  if (stage_in && (rc = grow_pinned(r.pin_in, r.pin_in_bytes, (size_t)row * src_rows))) return rc;
  if (stage_out && (rc = grow_pinned(r.pin_out, r.pin_out_bytes, (size_t)row * out_rows))) return rc;
  char* din = static_cast<char*>(r.dbuf);
  char* dout = din + (size_t)row * src_rows;
  char* pin = static_cast<char*>(r.pin_in);
  char* pout = static_cast<char*>(r.pin_out);
  CopyPool& pool = CopyPool::get();

  // sub-bands of >= 64 rows and >= 2 MB, at most 16 (measured on C2 with
  // pinned buffers: 1 -> 19.3, 4 -> 27.8, 8 -> 34.7, 16 -> 38.7,
  // 32 -> 35.5 Gpixel/s e2e); small images get one band
  static const int force_nb = [] {  // experiments: TMB_HOST_BANDS
    const char* v = getenv("TMB_HOST_BANDS");
    return v ? atoi(v) : 0;
  }();
  const int64_t img_bytes = row * out_rows;
  const int nb = force_nb > 0 ? std::min(std::min(force_nb, kMaxBands), out_rows)
                              : (int)std::max<int64_t>(1, std::min<int64_t>(
                                    {16, out_rows / 64, img_bytes / (2 << 20)}));
  int y[kMaxBands + 1], c[kMaxBands + 1];  // output sub-bands / source chunks (absolute rows)
  for (int b = 0; b <= nb; b++) {
    y[b] = ya + (int)((int64_t)out_rows * b / nb);
    c[b] = sa + (int)((int64_t)src_rows * b / nb);
  }
  // source chunk holding row `s` (absolute)
  auto chunk_of = [&](int s) {
    int ch = 0;
    while (ch + 1 < nb && c[ch + 1] <= s) ch++;
    return ch;
  };
  int next_filter = 0;
  double t_copy_in = 0.0, t_copy_out = 0.0;
  const double t_start = g_trace ? now_ms() : 0.0;
  auto issue_filters = [&](int chunks_ready) -> int {
    while (next_filter < nb) {
      const int b = next_filter;
      const int need = chunk_of(std::min(sb, y[b + 1] + halo) - 1);
      if (need >= chunks_ready) break;
      cudaStream_t fst = r.fs[b % kFilterStreams];
      cudaError_t e2 = cudaStreamWaitEvent(fst, r.ev_in[need], 0);
      if (e2 != cudaSuccess) return set_error(TM_ECUDA, "stream wait: %s", cudaGetErrorString(e2));
      int rc2 = tm_median2d_band(din, row, src_rows, y[b] - sa, y[b + 1] - y[b],
                                 dout + (size_t)(y[b] - ya) * row, row, a.width, a.channels,
                                 a.bits, a.k_w, a.k_h, a.variant, fst);
      if (rc2) return rc2;
      e2 = cudaEventRecord(r.ev_out[b], fst);
      if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(r.d2h, r.ev_out[b], 0);
      const int64_t n_rows = y[b + 1] - y[b];
      const char* from = dout + (size_t)(y[b] - ya) * row;
      if (e2 == cudaSuccess) {
        if (stage_out)
          e2 = cudaMemcpyAsync(pout + (size_t)(y[b] - ya) * row, from, (size_t)(n_rows * row),
                               cudaMemcpyDeviceToHost, r.d2h);
        else if (a.dst_pitch == row)
          e2 = cudaMemcpyAsync(a.dst + (int64_t)y[b] * row, from, (size_t)(n_rows * row),
                               cudaMemcpyDeviceToHost, r.d2h);
        else
          e2 = cudaMemcpy2DAsync(a.dst + (int64_t)y[b] * a.dst_pitch, a.dst_pitch, from, row, row,
                                 n_rows, cudaMemcpyDeviceToHost, r.d2h);
      }
      if (e2 == cudaSuccess) e2 = cudaEventRecord(r.ev_d2h[b], r.d2h);
      if (e2 != cudaSuccess) return set_error(TM_ECUDA, "D2H copy: %s", cudaGetErrorString(e2));
      next_filter++;
    }
    return TM_OK;
  };
  for (int b = 0; b < nb; b++) {
    const int64_t n_rows = c[b + 1] - c[b];
    char* to = din + (size_t)(c[b] - sa) * row;
    const char* from = a.src + (int64_t)c[b] * a.src_pitch;
    if (stage_in) {
      char* st = pin + (size_t)(c[b] - sa) * row;
      const double tc = g_trace ? now_ms() : 0.0;
      pool.copy2d(st, row, from, a.src_pitch, row, n_rows);  // overlaps the previous chunk's DMA
      if (g_trace) t_copy_in += now_ms() - tc;
      e = cudaMemcpyAsync(to, st, (size_t)(n_rows * row), cudaMemcpyHostToDevice, r.h2d);
    } else if (a.src_pitch == row) {
      e = cudaMemcpyAsync(to, from, (size_t)(n_rows * row), cudaMemcpyHostToDevice, r.h2d);
    } else {
      e = cudaMemcpy2DAsync(to, row, from, a.src_pitch, row, n_rows, cudaMemcpyHostToDevice, r.h2d);
    }
    if (e == cudaSuccess) e = cudaEventRecord(r.ev_in[b], r.h2d);
    if (e != cudaSuccess) return set_error(TM_ECUDA, "H2D copy: %s", cudaGetErrorString(e));
    if ((rc = issue_filters(b + 1))) return rc;
  }
  if ((rc = issue_filters(nb))) return rc;
  if (stage_out) {
    for (int b = 0; b < nb; b++) {
      e = cudaEventSynchronize(r.ev_d2h[b]);
      if (e != cudaSuccess) return set_error(TM_ECUDA, "kernel or copy failed: %s", cudaGetErrorString(e));
      const double tc = g_trace ? now_ms() : 0.0;
      pool.copy2d(a.dst + (int64_t)y[b] * a.dst_pitch, a.dst_pitch,
                  pout + (size_t)(y[b] - ya) * row, row, row, y[b + 1] - y[b]);
      if (g_trace) t_copy_out += now_ms() - tc;
    }
  }
  const double t_issued = g_trace ? now_ms() : 0.0;
  e = cudaStreamSynchronize(r.d2h);
  for (auto& st : r.fs)
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(r.h2d);
  if (e != cudaSuccess) return set_error(TM_ECUDA, "kernel failed: %s", cudaGetErrorString(e));
  if (g_trace)
    fprintf(stderr, "[tm_host] rows %d..%d bands %d stage_in %d stage_out %d: copy-in %.2f ms, "
            "copy-out %.2f ms, issued at %.2f ms, done at %.2f ms\n", ya, yb, nb, (int)stage_in,
            (int)stage_out, t_copy_in, t_copy_out, t_issued - t_start, now_ms() - t_start);
  return TM_OK;
}

// Output rows [ya, yb) on `device` in memory bands: each band's device
// buffers (its source rows with the k_h/2 halos + its output rows) stay within
// `budget` bytes (0 = half of the device's free memory) -- the reference's
// slice_budget banding (aware.py:455-463), exact for the same reason: every
// band re-reads its halo rows from the original image.
int host_range(const HostArgs& a, int device, int ya, int yb, int64_t budget = 0) {
  const int64_t row = (int64_t)a.width * a.channels * (a.bits / 8);
  const int halo = a.k_h / 2;
  if (budget <= 0 && device >= 0 && device < kMaxDev) {
    // already holding enough device memory for the whole range: one band
    const int64_t need = row * ((int64_t)std::min(a.height, yb + halo) - std::max(0, ya - halo) +
                                (yb - ya));
    std::lock_guard<std::mutex> g(g_dev[device].mu);
    if ((int64_t)g_dev[device].dbytes >= need) budget = need;
  }
  if (budget <= 0) {
    size_t fr = 0, tot = 0;
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) == cudaSuccess && cudaMemGetInfo(&fr, &tot) == cudaSuccess)
      budget = (int64_t)(fr / 2) + (int64_t)g_dev[device < kMaxDev && device >= 0 ? device : 0].dbytes;
    else
      cudaGetLastError();
    if (prev >= 0) cudaSetDevice(prev);
    if (budget <= 0) budget = (int64_t)1 << 30;
  }
  const int64_t per = budget / row;  // rows that fit
  // a budget below one output row plus its halos still works, one row per band
  // (like the reference, whose bands shrink to one tile row)
  const int64_t chunk = std::max<int64_t>(1, (per - 2 * halo) / 2);
  for (int y = ya; y < yb; y += (int)std::min<int64_t>(chunk, yb - y)) {
    const int rc = host_chunk(a, device, y, (int)std::min<int64_t>(yb, y + chunk));
    if (rc) return rc;
  }
  return TM_OK;
}

int check_host(const HostArgs& a) {
  if (a.bits != 8 && a.bits != 16 && a.bits != 32)
    return set_error(TM_ETYPE, "unsupported element width %d bits (expected 8, 16 or 32)", a.bits);
  if (a.width < 1 || a.height < 1)
    return set_error(TM_EINVAL, "expected a non-empty 2-D image, got %dx%d", a.width, a.height);
  if (!a.src || !a.dst) return set_error(TM_EINVAL, "null buffer");
  if (a.channels < 1 || a.channels > 65535) return set_error(TM_EINVAL, "bad channel count %d", a.channels);
  const int64_t row = (int64_t)a.width * a.channels * (a.bits / 8);
  if (a.src_pitch < row || a.dst_pitch < row) return set_error(TM_EINVAL, "pitch smaller than a row");
  // kernel sides / variant: validated by tm_median2d_band (same messages)
  if (tm_dispatch_query(a.bits, a.k_w, a.k_h, a.variant) == TM_KERNEL_NONE)
    return tm_median2d_band(a.src, a.src_pitch, a.height, 0, 0, a.dst, a.dst_pitch, a.width,
                            a.channels, a.bits, a.k_w, a.k_h, a.variant, nullptr);
  return TM_OK;
}

}  // namespace

extern "C" {

int tm_median2d_host(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                     int32_t width, int32_t height, int32_t channels, int32_t bits, int32_t k_w,
                     int32_t k_h, int32_t variant, int32_t device) {
  return tm_median2d_host_budget(src, src_pitch, dst, dst_pitch, width, height, channels, bits,
                                 k_w, k_h, variant, device, 0);
}

int tm_median2d_host_budget(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                            int32_t width, int32_t height, int32_t channels, int32_t bits,
                            int32_t k_w, int32_t k_h, int32_t variant, int32_t device,
                            int64_t device_budget) {
  const HostArgs a{static_cast<const char*>(src), src_pitch, static_cast<char*>(dst), dst_pitch,
                   width, height, channels, bits, k_w, k_h, variant};
  int rc = check_host(a);
  if (rc) return rc;
  if (device < 0 || device >= kMaxDev) return set_error(TM_EINVAL, "bad device %d", device);
  DeviceGuard guard;
  return host_range(a, device, 0, height, device_budget);
}

int tm_median2d_host_multi(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                           int32_t width, int32_t height, int32_t channels, int32_t bits,
                           int32_t k_w, int32_t k_h, int32_t variant, const int32_t* dev_ids,
                           int32_t n_dev) {
  const HostArgs a{static_cast<const char*>(src), src_pitch, static_cast<char*>(dst), dst_pitch,
                   width, height, channels, bits, k_w, k_h, variant};
  int rc = check_host(a);
  if (rc) return rc;
  if (n_dev < 1 || !dev_ids) return set_error(TM_EINVAL, "need at least one device");
  DeviceGuard guard;
  const int n = std::min(n_dev, height);
  if (n == 1) return host_range(a, dev_ids[0], 0, height);
  // balanced row bands (earlier devices get +1 row), one host thread each;
  // each device reads its own k_h/2 halo rows straight from the host image
  std::vector<int> rcs(n, TM_OK);
  std::vector<std::string> errs(n);
  std::vector<std::thread> th;
  for (int i = 0; i < n; i++) {
    const int base = height / n, extra = height % n;
    const int ya = i * base + std::min(i, extra), yb = ya + base + (i < extra ? 1 : 0);
    th.emplace_back([&, i, ya, yb] {
      rcs[i] = host_range(a, dev_ids[i], ya, yb);
      if (rcs[i]) errs[i] = tm_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int i = 0; i < n; i++)
    if (rcs[i]) return set_error(rcs[i], "device %d: %s", dev_ids[i], errs[i].c_str());
  return TM_OK;
}

int tm_median2d_host_frames(const void* src, int64_t src_pitch, int64_t src_frame_bytes,
                            void* dst, int64_t dst_pitch, int64_t dst_frame_bytes,
                            int32_t n_frames, int32_t width, int32_t height, int32_t channels,
                            int32_t bits, int32_t k_w, int32_t k_h, int32_t variant,
                            const int32_t* dev_ids, int32_t n_dev) {
  if (n_frames < 0) return set_error(TM_EINVAL, "bad frame count %d", n_frames);
  if (n_frames == 0) return TM_OK;
  const HostArgs a0{static_cast<const char*>(src), src_pitch, static_cast<char*>(dst), dst_pitch,
                    width, height, channels, bits, k_w, k_h, variant};
  int rc = check_host(a0);
  if (rc) return rc;
  const int64_t frame = (int64_t)height * std::max(src_pitch, dst_pitch);
  if (src_frame_bytes < (int64_t)height * src_pitch || dst_frame_bytes < (int64_t)height * dst_pitch)
    return set_error(TM_EINVAL, "frame stride smaller than a frame (%lld bytes)", (long long)frame);
  if (n_dev < 1 || !dev_ids) return set_error(TM_EINVAL, "need at least one device");
  DeviceGuard guard;
  // frames are independent: frame f goes to device dev_ids[f % n_dev], one
  // host thread per device, no communication ("batches of frames are split
  // across GPUs")
  const int n = std::min(n_dev, n_frames);
  std::vector<int> rcs(n, TM_OK);
  std::vector<std::string> errs(n);
  auto work = [&](int i) {
    for (int f = i; f < n_frames; f += n) {
      HostArgs a = a0;
      a.src += (int64_t)f * src_frame_bytes;
      a.dst += (int64_t)f * dst_frame_bytes;
      rcs[i] = host_range(a, dev_ids[i], 0, height);
      if (rcs[i]) {
        errs[i] = tm_last_error();
        return;
      }
    }
  };
  if (n == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int i = 0; i < n; i++) th.emplace_back(work, i);
    for (auto& t : th) t.join();
  }
  for (int i = 0; i < n; i++)
    if (rcs[i]) return set_error(rcs[i], "device %d: %s", dev_ids[i], errs[i].c_str());
  return TM_OK;
}

int tm_median2d_bands(void* const* band_buf, const int64_t* band_pitch, void* const* band_dst,
                      const int64_t* dst_pitch, const int32_t* band_rows, const int32_t* dev_ids,
                      int32_t n_bands, int32_t width, int32_t channels, int32_t bits, int32_t k_w,
                      int32_t k_h, int32_t variant, void* const* streams) {
  if (n_bands < 1 || !band_buf || !band_pitch || !band_dst || !dst_pitch || !band_rows || !dev_ids)
    return set_error(TM_EINVAL, "bad band arrays");
  const int halo = k_h / 2;
  const int esz = bits / 8;
  for (int i = 0; i < n_bands; i++) {
    if (band_rows[i] < 1) return set_error(TM_EINVAL, "band %d is empty", i);
    if (n_bands > 1 && band_rows[i] < halo)
      return set_error(TM_EINVAL, "band %d has %d rows, fewer than the %d-row halo", i,
                       band_rows[i], halo);
  }
  DeviceGuard guard;
  auto stream_of = [&](int i) { return streams ? static_cast<cudaStream_t>(streams[i]) : nullptr; };
  const int64_t row = (int64_t)width * channels * esz;
  cudaError_t e = cudaSuccess;
  // peer access between neighbouring devices (NVLink / NVSwitch); without it
  // the copies still work through the host
  for (int i = 0; i + 1 < n_bands && n_bands > 1; i++) {
    const int a = dev_ids[i], b = dev_ids[i + 1];
    if (a == b) continue;
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, b, a);
    if (ok && cudaSetDevice(b) == cudaSuccess) {
      cudaError_t pe = cudaDeviceEnablePeerAccess(a, 0);
      if (pe != cudaSuccess) cudaGetLastError();  // already enabled is fine
    }
    cudaDeviceCanAccessPeer(&ok, a, b);
    if (ok && cudaSetDevice(a) == cudaSuccess) {
      cudaError_t pe = cudaDeviceEnablePeerAccess(b, 0);
      if (pe != cudaSuccess) cudaGetLastError();
    }
  }
  // 1. every band's current contents are ready on its own stream
  std::vector<cudaEvent_t> ready(n_bands, nullptr), halo_done(n_bands, nullptr);
  auto cleanup = [&] {
    for (auto ev : ready)
      if (ev) cudaEventDestroy(ev);
    for (auto ev : halo_done)
      if (ev) cudaEventDestroy(ev);
  };
  for (int i = 0; i < n_bands && e == cudaSuccess; i++) {
    e = cudaSetDevice(dev_ids[i]);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&halo_done[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ready[i], stream_of(i));
  }
  // 2. halo rows: band i's top halo <- the last h rows of band i-1, its bottom
  //    halo <- the first h rows of band i+1 (peer copies on band i's stream)
  for (int i = 0; i < n_bands && e == cudaSuccess && halo > 0; i++) {
    e = cudaSetDevice(dev_ids[i]);
    char* base = static_cast<char*>(band_buf[i]);
    if (i > 0 && e == cudaSuccess) {
      const char* nb = static_cast<const char*>(band_buf[i - 1]);
      e = cudaStreamWaitEvent(stream_of(i), ready[i - 1], 0);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(base, band_pitch[i], nb + (int64_t)band_rows[i - 1] * band_pitch[i - 1],
                              band_pitch[i - 1], row, halo, cudaMemcpyDefault, stream_of(i));
    }
    if (i + 1 < n_bands && e == cudaSuccess) {
      const char* nb = static_cast<const char*>(band_buf[i + 1]);
      e = cudaStreamWaitEvent(stream_of(i), ready[i + 1], 0);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(base + (int64_t)(halo + band_rows[i]) * band_pitch[i], band_pitch[i],
                              nb + (int64_t)halo * band_pitch[i + 1], band_pitch[i + 1], row, halo,
                              cudaMemcpyDefault, stream_of(i));
    }
    if (e == cudaSuccess) e = cudaEventRecord(halo_done[i], stream_of(i));
  }
  if (e != cudaSuccess) {
    cleanup();
    return set_error(TM_ECUDA, "halo exchange: %s", cudaGetErrorString(e));
  }
  // 3. a neighbour's rows must not change until the copies reading them land
  for (int i = 0; i < n_bands && e == cudaSuccess; i++) {
    e = cudaSetDevice(dev_ids[i]);
    if (i > 0 && e == cudaSuccess) e = cudaStreamWaitEvent(stream_of(i), halo_done[i - 1], 0);
    if (i + 1 < n_bands && e == cudaSuccess) e = cudaStreamWaitEvent(stream_of(i), halo_done[i + 1], 0);
  }
  // 4. filter every band on its device: reads clamp only at the true image edges
  int rc = TM_OK;
  for (int i = 0; i < n_bands && e == cudaSuccess && rc == TM_OK; i++) {
    e = cudaSetDevice(dev_ids[i]);
    if (e != cudaSuccess) break;
    const char* base = static_cast<const char*>(band_buf[i]);
    const int top = (i > 0) ? halo : 0;
    const int bot = (i + 1 < n_bands) ? halo : 0;
    const char* s = base + (int64_t)(halo - top) * band_pitch[i];
    rc = tm_median2d_band(s, band_pitch[i], top + band_rows[i] + bot, top, band_rows[i], band_dst[i],
                          dst_pitch[i], width, channels, bits, k_w, k_h, variant, stream_of(i));
  }
  if (e == cudaSuccess) {
    // events may be destroyed once recorded work is enqueued
    cleanup();
  } else {
    cleanup();
    return set_error(TM_ECUDA, "band filter: %s", cudaGetErrorString(e));
  }
  return rc;
}

void* tm_host_alloc(int64_t bytes) {
  if (bytes < 0) return nullptr;
  return PinnedPool::get().alloc((size_t)bytes);
}

int tm_host_free(void* p) {
  if (!PinnedPool::get().release(p)) return set_error(TM_EINVAL, "not a tm_host_alloc block");
  return TM_OK;
}

}  // extern "C"
