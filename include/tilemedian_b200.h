/*
 * tilemedian_b200.h -- C ABI of the B200 (sm_100a) hierarchical-tiling median
 * filter.  Drop-in boundary for the reference package's median-filter entry
 * points (reference: /root/reference/pkg/src/tilemedian/engine.py):
 *
 *   tm_median2d        <- filter_image(image, k, variant)      engine.py:29-52
 *   tm_median2d_rect   <- filter_image(image, KernelSpec(..))  engine.py:24-25, 43-44
 *   tm_median2d_planes <- filter_planes(image (H,W,C), k)      engine.py:55-64
 *   tm_median2d_band   <- the per-band work of the reference's banded engines
 *                         (oblivious.py:351-394 bands of tile rows, aware.py:
 *                         455-491 bands re-reading +-k/2 halo rows): one band
 *                         of output rows from a source that carries its halo
 *   tm_median2d_host   <- filter_image on host (numpy) buffers, copies included
 *   tm_median2d_host_multi <- filter_image(..., devices=[...]): one row band
 *                         per GPU, each re-reading its k_h/2 halo rows (the
 *                         reference's banding, aware.py:455-491)
 *   tm_median2d_host_frames <- a batch of frames (filter_frames): frames split
 *                         across the GPUs, no communication
 *   tm_median2d_bands  <- the same banding on device-resident bands: halo rows
 *                         exchanged between the GPUs (peer copies over NVLink)
 *   tm_host_alloc/free <- the reference returns a fresh host array
 *                         (oblivious.py:349); the drop-in returns it in pinned
 *                         memory so the device-to-host copy runs at full speed
 *   tm_dispatch_query  <- pick_variant(k)                       engine.py:22-26
 *
 * Semantics (bit-exact with reference.py:26-43): out[y][x] is the rank
 * (k_w*k_h+1)/2 (1-based) value of the k_h x k_w window centred on (x, y),
 * window coordinates clamped to the image (replicate borders; there is no
 * border argument).  Sides odd and >= 3.  bits in {8, 16, 32}
 * (unsigned).  Pitches are in BYTES.  Device pointers, caller-owned buffers,
 * stream-ordered (`stream` is a cudaStream_t, NULL = legacy default stream).
 * Output buffers must not alias inputs.
 *
 * Return codes: TM_OK, or TM_EINVAL (bad argument: Python raises ValueError),
 * TM_ETYPE (unsupported element width: TypeError), TM_ECUDA (CUDA error:
 * RuntimeError).  tm_last_error() returns the calling thread's last message.
 * All functions are thread-safe; the dispatch table is immutable.
 */
#ifndef TILEMEDIAN_B200_H
#define TILEMEDIAN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* variant argument: VARIANTS = ("auto", "oblivious", "aware", "oracle"), engine.py:18 */
enum {
  TM_VARIANT_AUTO = 0,
  TM_VARIANT_OBLIVIOUS = 1,
  TM_VARIANT_AWARE = 2,
  TM_VARIANT_ORACLE = 3
};

/* kernels tm_dispatch_query can report */
enum {
  TM_KERNEL_NONE = 0,
  TM_KERNEL_OBLIVIOUS = 1, /* register-resident selection network, variant (1) */
  TM_KERNEL_MULTIPASS = 2, /* the reference's multi-pass aware engine on the GPU (aware.py:437-492) */
  TM_KERNEL_SELECT = 3,    /* brute-force per-pixel radix selection ("oracle") */
  TM_KERNEL_HISTOGRAM = 4, /* 8-bit sliding column histograms: variant (2) for uint8 */
  TM_KERNEL_RANK = 5,      /* 16/32-bit coarse + candidate-key histogram sweeps: variant (2) */
  TM_KERNEL_MED3 = 6       /* k = 3: register sliding window, shared column sorts: variant (1) */
};

enum { TM_OK = 0, TM_EINVAL = 1, TM_ETYPE = 2, TM_ECUDA = 3 };

/* Square k x k median of a (height x width) device image. */
int tm_median2d(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                int32_t width, int32_t height, int32_t bits, int32_t k,
                int32_t variant, void* stream);

/* Rectangular k_w x k_h window. */
int tm_median2d_rect(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                     int32_t width, int32_t height, int32_t bits, int32_t k_w,
                     int32_t k_h, int32_t variant, void* stream);

/* Interleaved (height, width, channels) image, every channel filtered
 * separately (one launch for all planes). */
int tm_median2d_planes(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                       int32_t width, int32_t height, int32_t channels, int32_t bits,
                       int32_t k, int32_t variant, void* stream);

/* General band form.  `src` holds src_rows rows; output rows
 * [out_row0, out_row0 + out_rows) of that source are written to dst rows
 * [0, out_rows).  Window reads clamp to the source's rows, so a band whose
 * source includes +-k_h/2 halo rows from its neighbours (and clamps only at
 * the true image edges) is bit-identical to the whole-image result. */
int tm_median2d_band(const void* src, int64_t src_pitch, int32_t src_rows,
                     int32_t out_row0, int32_t out_rows, void* dst, int64_t dst_pitch,
                     int32_t width, int32_t channels, int32_t bits, int32_t k_w,
                     int32_t k_h, int32_t variant, void* stream);

/* Host buffers: copies in, filters on `device`, copies out, synchronises. */
int tm_median2d_host(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                     int32_t width, int32_t height, int32_t channels, int32_t bits,
                     int32_t k_w, int32_t k_h, int32_t variant, int32_t device);

/* tm_median2d_host with the device memory held per call bounded by
 * device_budget bytes (0 = half the free memory): the image is processed in
 * row bands whose buffers (source rows with their k_h/2 halos + output rows)
 * fit (at least one output row per band) -- the reference's slice_budget
 * banding (aware.py:455-463); the result does not depend on the budget. */
int tm_median2d_host_budget(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                            int32_t width, int32_t height, int32_t channels, int32_t bits,
                            int32_t k_w, int32_t k_h, int32_t variant, int32_t device,
                            int64_t device_budget);

/* Host buffers split into n_dev balanced row bands, one per device in
 * dev_ids, filtered concurrently (a repeated ordinal runs its bands one after
 * the other); every device copies its
 * own band plus k_h/2 halo rows from the host image, so the result is
 * bit-identical to tm_median2d_host.  Synchronises. */
int tm_median2d_host_multi(const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                           int32_t width, int32_t height, int32_t channels, int32_t bits,
                           int32_t k_w, int32_t k_h, int32_t variant, const int32_t* dev_ids,
                           int32_t n_dev);

/* A batch of n_frames independent host images (frame f at src + f *
 * src_frame_bytes, output at dst + f * dst_frame_bytes), frame f filtered on
 * device dev_ids[f % n_dev]; devices run concurrently, no communication.
 * Synchronises. */
int tm_median2d_host_frames(const void* src, int64_t src_pitch, int64_t src_frame_bytes,
                            void* dst, int64_t dst_pitch, int64_t dst_frame_bytes,
                            int32_t n_frames, int32_t width, int32_t height, int32_t channels,
                            int32_t bits, int32_t k_w, int32_t k_h, int32_t variant,
                            const int32_t* dev_ids, int32_t n_dev);

/* Device-resident row bands of one image, band i (rows top to bottom) on
 * device dev_ids[i].  band_buf[i] holds h = k_h/2 halo rows, then its
 * band_rows[i] rows, then h halo rows (pitch band_pitch[i] bytes); the halo
 * rows are filled here from the neighbouring bands (peer copies, NVLink when
 * peer access is available) -- the first band's top and the last band's
 * bottom halo are neither written nor read.  Output band i goes to
 * band_dst[i] (band_rows[i] rows, pitch dst_pitch[i]) on streams[i] (NULL
 * array = default streams); every band needs >= h rows when n_bands > 1.
 * Stream-ordered; bit-identical to filtering the whole image on one GPU. */
int tm_median2d_bands(void* const* band_buf, const int64_t* band_pitch, void* const* band_dst,
                      const int64_t* dst_pitch, const int32_t* band_rows, const int32_t* dev_ids,
                      int32_t n_bands, int32_t width, int32_t channels, int32_t bits,
                      int32_t k_w, int32_t k_h, int32_t variant, void* const* streams);

/* Pinned, portable host memory from a size-bucketed cache (NULL on failure);
 * tm_host_free returns a block to the cache. */
void* tm_host_alloc(int64_t bytes);
int tm_host_free(void* p);

/* Which kernel serves (bits, k_w, k_h, variant); TM_KERNEL_NONE if invalid. */
int tm_dispatch_query(int32_t bits, int32_t k_w, int32_t k_h, int32_t variant);
const char* tm_kernel_name(int32_t kernel);

/* Diagnostics (sweeps, tests): force the calling thread's launches onto one
 * kernel when it supports (bits, k); 0 restores the dispatch table.  Returns
 * the previous setting.  Results do not change -- every kernel is exact. */
int tm_force_kernel(int32_t kernel);

/* Number of kernel launches issued by this process so far (all entry points). */
int64_t tm_launch_count(void);

const char* tm_last_error(void);
const char* tm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TILEMEDIAN_B200_H */
