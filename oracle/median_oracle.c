/*
 * median_oracle.c -- CPU restatement of the reference's brute-force median
 * filter.  TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs, as the checker or the
 * reported CPU baseline.  The product path never calls into this library.
 *
 * Follows /root/reference/pkg/src/tilemedian/reference.py:26-43
 * (oracle_median_filter):
 *   - edge-replicated borders (np.pad mode="edge", reference.py:37-38): every
 *     window coordinate is clamped into [0, W-1] x [0, H-1];
 *   - the window is k_h x k_w (KernelSpec, geometry.py:25-58), odd sides;
 *   - output = the rank-(k_w*k_h+1)/2 value (1-based) of the window
 *     (np.partition at rank-1, reference.py:41-43).
 * Per pixel it gathers the clamped window and selects the rank with
 *   - a 256-bin histogram for 8-bit data, and
 *   - an in-place quickselect for 16/32-bit data.
 * Rows are split across `threads` POSIX threads (row bands); output is
 * independent of the thread count.
 *
 * "Band" form: the caller may pass a row range [y0, y1) so a large image can
 * be checked (or timed) a band at a time; clamping still uses the full image
 * height, exactly like the banded oracle of SURVEY.md section 7 step 1.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const void *src;
  void *dst;
  int64_t src_pitch, dst_pitch; /* elements */
  int width, height, bits, kw, kh;
  int y0, y1;
} job_t;

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

#define DEFINE_SELECT(T, NAME)                                               \
  static T NAME(T *a, int n, int rank) {                                     \
    int lo = 0, hi = n - 1;                                                  \
    while (hi > lo) {                                                        \
      int mid = lo + ((hi - lo) >> 1);                                       \
      T x = a[lo], y = a[mid], z = a[hi], p;                                 \
      /* median of three as pivot */                                         \
      if (x < y) p = (y < z) ? y : ((x < z) ? z : x);                        \
      else p = (x < z) ? x : ((y < z) ? z : y);                              \
      int i = lo, j = hi;                                                    \
      while (i <= j) {                                                       \
        while (a[i] < p) i++;                                                \
        while (p < a[j]) j--;                                                \
        if (i <= j) { T t = a[i]; a[i] = a[j]; a[j] = t; i++; j--; }         \
      }                                                                      \
      if (rank <= j) hi = j;                                                 \
      else if (rank >= i) lo = i;                                            \
      else return a[rank];                                                   \
    }                                                                        \
    return a[rank];                                                          \
  }

DEFINE_SELECT(uint16_t, select_u16)
DEFINE_SELECT(uint32_t, select_u32)

static void run_u8(const job_t *jb) {
  const uint8_t *src = (const uint8_t *)jb->src;
  uint8_t *dst = (uint8_t *)jb->dst;
  const int hw = jb->kw / 2, hh = jb->kh / 2;
  const int rank = (jb->kw * jb->kh + 1) / 2; /* 1-based */
  int *xs = (int *)malloc(sizeof(int) * jb->kw);
  for (int y = jb->y0; y < jb->y1; y++) {
    for (int x = 0; x < jb->width; x++) {
      uint32_t hist[256];
      memset(hist, 0, sizeof(hist));
      for (int dx = 0; dx < jb->kw; dx++) xs[dx] = clampi(x + dx - hw, 0, jb->width - 1);
      for (int dy = -hh; dy <= hh; dy++) {
        const uint8_t *row = src + (int64_t)clampi(y + dy, 0, jb->height - 1) * jb->src_pitch;
        for (int dx = 0; dx < jb->kw; dx++) hist[row[xs[dx]]]++;
      }
      int acc = 0, v = 0;
      for (; v < 256; v++) {
        acc += (int)hist[v];
        if (acc >= rank) break;
      }
      dst[(int64_t)y * jb->dst_pitch + x] = (uint8_t)v;
    }
  }
  free(xs);
}

#define DEFINE_RUN(T, NAME, SEL)                                                      \
  static void NAME(const job_t *jb) {                                                 \
    const T *src = (const T *)jb->src;                                                \
    T *dst = (T *)jb->dst;                                                            \
    const int hw = jb->kw / 2, hh = jb->kh / 2, n = jb->kw * jb->kh;                 \
    const int rank0 = (n + 1) / 2 - 1;                                                \
    T *win = (T *)malloc(sizeof(T) * (size_t)n);                                      \
    int *xs = (int *)malloc(sizeof(int) * jb->kw);                                    \
    for (int y = jb->y0; y < jb->y1; y++) {                                           \
      for (int x = 0; x < jb->width; x++) {                                           \
        for (int dx = 0; dx < jb->kw; dx++) xs[dx] = clampi(x + dx - hw, 0, jb->width - 1); \
        int m = 0;                                                                    \
        for (int dy = -hh; dy <= hh; dy++) {                                          \
          const T *row = src + (int64_t)clampi(y + dy, 0, jb->height - 1) * jb->src_pitch; \
          for (int dx = 0; dx < jb->kw; dx++) win[m++] = row[xs[dx]];                 \
        }                                                                             \
        dst[(int64_t)y * jb->dst_pitch + x] = SEL(win, n, rank0);                     \
      }                                                                               \
    }                                                                                 \
    free(win);                                                                        \
    free(xs);                                                                         \
  }

DEFINE_RUN(uint16_t, run_u16, select_u16)
DEFINE_RUN(uint32_t, run_u32, select_u32)

static void *worker(void *arg) {
  const job_t *jb = (const job_t *)arg;
  if (jb->bits == 8) run_u8(jb);
  else if (jb->bits == 16) run_u16(jb);
  else run_u32(jb);
  return NULL;
}

/*
 * Median-filter rows [y0, y1) of a (height x width) image.  Pitches are in
 * elements.  Returns 0 on success, -1 on a bad argument.
 */
int oracle_median2d(const void *src, int64_t src_pitch, void *dst, int64_t dst_pitch,
                    int width, int height, int bits, int kw, int kh, int y0, int y1,
                    int threads) {
  if (!src || !dst || width < 1 || height < 1) return -1;
  if (bits != 8 && bits != 16 && bits != 32) return -1;
  if (kw < 1 || kh < 1 || !(kw & 1) || !(kh & 1)) return -1;
  if (y0 < 0 || y1 > height || y0 > y1) return -1;
  if (threads < 1) threads = 1;
  int rows = y1 - y0;
  if (threads > rows) threads = rows > 0 ? rows : 1;
  job_t *jobs = (job_t *)calloc((size_t)threads, sizeof(job_t));
  pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; t++) {
    job_t *jb = &jobs[t];
    jb->src = src; jb->dst = dst;
    jb->src_pitch = src_pitch; jb->dst_pitch = dst_pitch;
    jb->width = width; jb->height = height; jb->bits = bits; jb->kw = kw; jb->kh = kh;
    jb->y0 = y0 + (int)((int64_t)rows * t / threads);
    jb->y1 = y0 + (int)((int64_t)rows * (t + 1) / threads);
  }
  if (threads == 1) {
    worker(&jobs[0]);
  } else {
    for (int t = 0; t < threads; t++) pthread_create(&tids[t], NULL, worker, &jobs[t]);
    for (int t = 0; t < threads; t++) pthread_join(tids[t], NULL);
  }
  free(jobs);
  free(tids);
  return 0;
}
